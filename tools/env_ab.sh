#!/bin/bash
# One planner knob over its values, same box, alternating processes:
#   VAR=PMB_SCAN_TAILCLAIM VALUES="0 32 64" AB_CONFIGS="syn20k syn20k@512" tools/env_ab.sh
# (config@N: a batch of N chromosomes; value "auto" = the knob unset)
mkdir -p gpurun_out
for c in ${AB_CONFIGS:-syn20k syn20k@512 syn5k sweep:200 pmed40}; do
  cfg=${c%@*}; cnt=""; [ "$c" != "$cfg" ] && cnt=${c#*@}
  for r in 1 2; do
    for v in $VALUES; do
      if [ "$v" = auto ]; then unset $VAR; else export $VAR=$v; fi
      echo "$VAR=$v $c: $(TE_COUNT=$cnt timeout 300 python tools/time_eval.py $cfg ${AB_KIND:-scan} 10 auto 1 2>&1 | tail -1)"
      unset $VAR
    done
  done
done > gpurun_out/env_ab.log 2>&1
cat gpurun_out/env_ab.log
