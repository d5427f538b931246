#!/bin/bash
# same-box A/B/C: current build vs libpmedian_b200_ab.so (HEAD) vs libpmedian_b200_q2.so, alternating processes
mkdir -p gpurun_out
for c in ${AB_CONFIGS:-syn20k pmed40 syn5k}; do
  for r in 1 2 3; do
    echo "$c new: $(timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
    echo "$c old: $(PMB_LIBRARY=$PWD/paper_1610_10061_b200/libpmedian_b200_ab.so timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
    echo "$c q2:  $(PMB_LIBRARY=$PWD/paper_1610_10061_b200/libpmedian_b200_q2.so timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
  done
done > gpurun_out/ab3_time.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > gpurun_out/ab3_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/ab3_parity.log
cat gpurun_out/ab3_time.log; tail -n 2 gpurun_out/ab3_parity.log
