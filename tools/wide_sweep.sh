#!/bin/bash
# K2 many-warp variant (plan_scan default for long segments) vs the 16-warp shape (PMB_SCAN_WIDE=0)
for r in 1 2; do
  for c in ${CFGS:-syn20k}; do
    echo "wide: $(timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
    echo "16w:  $(PMB_SCAN_WIDE=0 timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
  done
done
