#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "parity or ingest" 2>&1 | tail -1
python tools/prof_eval.py syn20k scan 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:'k_build_rows' python tools/prof_eval.py syn20k scan 1 2>&1 | grep -E "gpu__time_duration|inst_exec" | head -4
