#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu -k "ga or island or run_ga or baseline or cpp or cli or orlib" > gpurun_out/ga_pipe_pytest.log 2>&1; tail -2 gpurun_out/ga_pipe_pytest.log
timeout 300 ./tests/cpp/_ref/acceptance | head -6
bash tools/build_ab.sh HEAD > /dev/null 2>&1 || echo "ab build failed (no nvcc?)"
AB=paper_1610_10061_b200/libpmedian_b200_ab.so
for r in 1 2; do
  echo "new: $(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed40 20 reference 2>&1 | tail -1)"
  echo "old: $(PMB_LIBRARY=$AB PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed40 20 reference 2>&1 | tail -1)"
  echo "new: $(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed40 20 device 2>&1 | tail -1)"
  echo "old: $(PMB_LIBRARY=$AB PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed40 20 device 2>&1 | tail -1)"
  echo "new: $(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed1 20 reference 2>&1 | tail -1)"
  echo "old: $(PMB_LIBRARY=$AB PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py pmed1 20 reference 2>&1 | tail -1)"
  echo "new: $(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py syn20k 10 reference 2>&1 | tail -1)"
  echo "old: $(PMB_LIBRARY=$AB PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py syn20k 10 reference 2>&1 | tail -1)"
done
