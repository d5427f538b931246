#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu -k "parity or cpp" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-ga > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for c in syn5k pmed40; do timeout 600 python bench.py --config $c --no-ga --no-cpu-baseline > gpurun_out/bench_$c.json 2>> gpurun_out/bench.err; done
