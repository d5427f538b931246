#!/bin/bash
# Cooperative-tail A/B: "log2(lanes per client) threshold" pairs (PMB_SCAN_COOPSEG, PMB_SCAN_COOP)
mkdir -p gpurun_out
for c in syn20k syn20k@512 syn5k sweep:200 sweep:1000 pmed40; do
  cfg=${c%@*}; cnt=""; [ "$c" != "$cfg" ] && cnt=${c#*@}
  for r in 1 2; do
    for v in "0 auto" "5 auto" "5 32" "4 32" "3 32"; do
      set -- $v
      export PMB_SCAN_COOPSEG=$1
      [ "$2" = auto ] && unset PMB_SCAN_COOP || export PMB_SCAN_COOP=$2
      echo "seg=$1 coop=$2 $c: $(TE_COUNT=$cnt timeout 300 python tools/time_eval.py $cfg scan 10 auto 1 2>&1 | tail -1)"
    done
    unset PMB_SCAN_COOPSEG PMB_SCAN_COOP
  done
done > gpurun_out/seg_ab.log 2>&1
cat gpurun_out/seg_ab.log
