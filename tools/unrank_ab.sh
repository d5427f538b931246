#!/bin/bash
# reference-exact population draw: log-guided k_unrank_log vs the lane-group probe (PMB_UNRANK=probe)
timeout 900 python -m pytest tests -x -q -m gpu -k "run_ga or evolve or draw or rank" > gpurun_out/ua_pytest.log 2>&1; tail -1 gpurun_out/ua_pytest.log
for r in 1 2; do for c in pmed40 pmed1; do
  echo "log:   $(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py $c 20 reference 2>&1 | tail -1)"
  echo "probe: $(PMB_UNRANK=probe PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py $c 20 reference 2>&1 | tail -1)"
done; done
python tools/prof_ga.py pmed40 3 reference > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_unrank" -c 4 python tools/prof_ga.py pmed40 3 reference 2>&1 | grep -E "k_unrank|duration" | head -8
