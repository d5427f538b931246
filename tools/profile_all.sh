#!/bin/bash
# One ncu --set full capture of the first launch of every library kernel (tools/prof_all.py).
mkdir -p gpurun_out
timeout 600 python tools/prof_all.py > gpurun_out/pa_plain.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on --kernel-id ::regex:^k_:1 \
  -o gpurun_out/all_kernels -f python tools/prof_all.py > gpurun_out/pa_ncu.log 2>&1
tail -3 gpurun_out/pa_plain.log; tail -3 gpurun_out/pa_ncu.log
