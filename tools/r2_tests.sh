#!/bin/bash
# GPU suite + the reference's acceptance gate on the compat headers (output kept).
set -u
mkdir -p gpurun_out
timeout 300 ./tests/cpp/_ref/acceptance > gpurun_out/acceptance.log 2>&1; echo "acceptance rc=$?" >> gpurun_out/acceptance.log
timeout 300 ./tests/cpp/_ref/ref_tests > gpurun_out/ref_tests.log 2>&1; echo "ref_tests rc=$?" >> gpurun_out/ref_tests.log
( time timeout 1800 python -m pytest tests -q -m gpu --durations=25 ${PYTEST_ARGS:-} ) > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat gpurun_out/acceptance.log; tail -4 gpurun_out/ref_tests.log; tail -40 gpurun_out/pytest_gpu.log
