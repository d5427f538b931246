#!/bin/bash
# Same-box timing of several library variants (PMB_LIBRARY), alternating processes:
#   VARIANTS="cur nosplit ab" AB_CONFIGS="syn20k pmed40" tools/ab_multi.sh
mkdir -p gpurun_out
for c in ${AB_CONFIGS:-syn20k pmed40 syn5k}; do
  for r in 1 2; do
    for v in ${VARIANTS:-cur ab}; do
      if [ "$v" = cur ]; then lib=""; else lib=paper_1610_10061_b200/libpmedian_b200_$v.so; fi
      echo "$v: $(PMB_LIBRARY=$lib timeout 300 python tools/time_eval.py $c ${AB_KIND:-scan} 10 auto 1 2>&1 | tail -1)"
    done
  done
done > gpurun_out/ab_multi.log 2>&1
cat gpurun_out/ab_multi.log
