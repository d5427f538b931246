#!/bin/bash
set -u
bash tools/gpu_round.sh
timeout 600 python bench.py --config syn5k --no-ga > gpurun_out/bench_syn5k.json 2>>gpurun_out/bench.err
timeout 600 python bench.py --config pmed40 --no-ga > gpurun_out/bench_pmed40.json 2>>gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash tools/profile_round.sh
