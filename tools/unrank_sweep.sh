#!/bin/bash
# k_unrank lanes-per-chromosome sweep at the paper's GA shape (reference-exact population draw)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "run_ga or evolve or draw or rank" > gpurun_out/unrank_pytest.log 2>&1; tail -2 gpurun_out/unrank_pytest.log
for S in 32 16 8 auto; do
  if [ $S = auto ]; then unset PMB_UNRANK_S; else export PMB_UNRANK_S=$S; fi
  echo "S=$S pmed40: $(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed40 20 reference 2>&1 | tail -1)"
  echo "S=$S pmed1: $(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed1 20 reference 2>&1 | tail -1)"
done
