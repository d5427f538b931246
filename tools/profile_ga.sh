#!/bin/bash
# GA launch list at the paper's Table-1 shape (pmed40 size, nb=60, nt=256): per-kernel share of a generation.
mkdir -p gpurun_out
G="python tools/prof_ga.py ${CFG:-pmed40} 5 ${POP:-reference}"
$G > gpurun_out/ga_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ga_launches.csv $G > gpurun_out/ga_ncu.log 2>&1
python tools/launch_table.py gpurun_out/ga_launches.csv "$G" > gpurun_out/ga_launches.md
cat gpurun_out/ga_plain.log; cat gpurun_out/ga_launches.md
