#!/bin/bash
# Cooperative-tail threshold (PMB_SCAN_COOP; auto = plan_scan's rule) on full
# batches and shard-sized ones (TE_COUNT), same box, alternating processes.
mkdir -p gpurun_out
for c in ${AB_CONFIGS:-syn20k syn20k@512 syn5k sweep:50 sweep:200 sweep:500 pmed40}; do
  cfg=${c%@*}; cnt=""; [ "$c" != "$cfg" ] && cnt=${c#*@}
  for r in 1 2; do
    for v in ${VALUES:-auto 0 4 8 12}; do
      if [ "$v" = auto ]; then unset PMB_SCAN_COOP; else export PMB_SCAN_COOP=$v; fi
      echo "coop=$v $c: $(TE_COUNT=$cnt timeout 300 python tools/time_eval.py $cfg ${AB_KIND:-scan} 10 auto 1 2>&1 | tail -1)"
      unset PMB_SCAN_COOP
    done
  done
done > gpurun_out/coop_ab.log 2>&1
cat gpurun_out/coop_ab.log
