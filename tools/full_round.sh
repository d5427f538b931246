#!/bin/bash
# Round validation: GPU tests, smoke, bench lines (syn20k with GA, syn5k, pmed40, reference arm).
# (ncu captures are separate calls: tools/profile_round.sh, tools/profile_all.sh -- the
# gpurun_out/ copy-back is capped at 64 MiB.)
set -u
bash tools/gpu_round.sh
timeout 600 python bench.py --config syn5k --no-ga > gpurun_out/bench_syn5k.json 2>>gpurun_out/bench.err
timeout 600 python bench.py --config pmed40 --no-ga > gpurun_out/bench_pmed40.json 2>>gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
