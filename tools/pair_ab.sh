#!/bin/bash
# Column-pair appends in the 24-warp K2 (plan_scan's m >= 75 p rule) against
# PMB_SCAN_PAIR=0 / =1, same box, alternating processes.
mkdir -p gpurun_out
for c in ${AB_CONFIGS:-syn20k sweep:50 sweep:100 sweep:200 sweep:500 sweep:1000}; do
  for r in 1 2; do
    for v in auto 0 1; do
      if [ "$v" = auto ]; then unset PMB_SCAN_PAIR; else export PMB_SCAN_PAIR=$v; fi
      echo "pair=$v $c: $(timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
    done
    unset PMB_SCAN_PAIR
  done
done > gpurun_out/pair_ab.log 2>&1
cat gpurun_out/pair_ab.log
