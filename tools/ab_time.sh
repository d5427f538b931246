#!/bin/bash
# same-box A/B: current build vs libpmedian_b200_ab.so (tools/build_ab.sh), alternating processes
mkdir -p gpurun_out
AB=paper_1610_10061_b200/libpmedian_b200_ab.so
for c in ${AB_CONFIGS:-syn20k pmed40 syn5k}; do
  for r in 1 2; do
    echo "new: $(timeout 300 python tools/time_eval.py $c ${AB_KIND:-scan} 10 auto 1 2>&1 | tail -1)"
    echo "old: $(PMB_LIBRARY=$AB timeout 300 python tools/time_eval.py $c ${AB_KIND:-scan} 10 auto 1 2>&1 | tail -1)"
  done
done > gpurun_out/ab_time.log 2>&1
cat gpurun_out/ab_time.log
