#!/bin/bash
# same-box A/B of the current build vs libpmedian_b200_ab.so: K2 kernel times and GA gens/s
mkdir -p gpurun_out
AB=paper_1610_10061_b200/libpmedian_b200_ab.so
for r in 1 2; do
  for c in syn20k pmed40 syn5k; do
    echo "new: $(timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
    echo "old: $(PMB_LIBRARY=$AB timeout 300 python tools/time_eval.py $c scan 10 auto 1 2>&1 | tail -1)"
  done
  echo "new: $(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed40 20 reference 2>&1 | tail -1)"
  echo "old: $(PMB_LIBRARY=$AB PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed40 20 reference 2>&1 | tail -1)"
  echo "new: $(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py syn20k 10 reference 2>&1 | tail -1)"
  echo "old: $(PMB_LIBRARY=$AB PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py syn20k 10 reference 2>&1 | tail -1)"
done > gpurun_out/ab_ga.log 2>&1
cat gpurun_out/ab_ga.log
