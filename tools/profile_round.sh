#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench run + full captures of K2, K2b, K1.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ga"
$B > gpurun_out/b_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
python tools/prof_eval.py syn20k scan 2 > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'^k_scan$' -c 1 -o gpurun_out/k2_scan_syn20k -f python tools/prof_eval.py syn20k scan 2 > gpurun_out/ncu1.log 2>&1
python tools/prof_eval.py syn5k gather 2 > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'^k_gather$' -c 1 -o gpurun_out/k2b_gather_syn5k -f python tools/prof_eval.py syn5k gather 2 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_build_rows' -c 1 -o gpurun_out/k1_build_syn20k -f python tools/prof_eval.py syn20k scan 1 > gpurun_out/ncu3.log 2>&1
for f in gpurun_out/ncu1.log gpurun_out/ncu2.log gpurun_out/ncu3.log gpurun_out/ncu_launch.log; do tail -n 1 $f; done
