#!/bin/bash
# scan-kernel experiment: parity tests + timings of the current build
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
for c in syn20k pmed40 syn5k; do timeout 300 python tools/time_eval.py $c scan 10 auto 3; done > gpurun_out/ab_time.log 2>&1
tail -2 gpurun_out/ab_pytest.log; cat gpurun_out/ab_time.log
