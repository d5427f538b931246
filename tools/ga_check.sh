#!/bin/bash
# GA kernels: parity tests, then generation rates at the paper's shape and pmed1's
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "${PYTEST_K:-run_ga or evolve or draw or rank or island}" > gpurun_out/ga_pytest.log 2>&1; tail -2 gpurun_out/ga_pytest.log
for c in pmed40 pmed1 syn20k; do
  for pop in reference device; do
    [ $c = syn20k ] && [ $pop = reference ] && continue
    echo "$(PROF_GA_REPS=2 timeout 300 python tools/prof_ga.py $c ${GENS:-20} $pop 2>&1 | tail -1)"
  done
done
