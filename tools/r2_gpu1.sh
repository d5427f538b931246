#!/bin/bash
# Round-2 validation call: GPU suite, smoke, bench (ours + reference arm), ncu of K2.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc >> gpurun_out/lscpu.txt; free -g >> gpurun_out/lscpu.txt
( time timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} ) > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/prof_eval.py syn20k scan 2 > gpurun_out/p1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^k_scan$' -c 1 -o gpurun_out/k2_scan_syn20k -f python tools/prof_eval.py syn20k scan 2 > gpurun_out/ncu1.log 2>&1 && \
python tools/ncu_to_json.py gpurun_out/k2_scan_syn20k.ncu-rep k_scan syn20k > gpurun_out/ncu1_json.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -c 600 gpurun_out/bench.json; tail -5 gpurun_out/bench.err; tail -c 300 gpurun_out/bench_ref.json; tail -2 gpurun_out/ncu1_json.log
