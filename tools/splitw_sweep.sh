#!/bin/bash
# K2 24-warp variant vs the 16-warp shapes (PMB_SCAN_WIDE=0) at the split-segment configs
for r in 1 2; do for c in ${CFGS:-pmed40 syn5k}; do
  echo "wide: $(timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
  echo "16w:  $(PMB_SCAN_WIDE=0 timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
done; done
