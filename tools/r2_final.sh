#!/bin/bash
# Round-2 final evidence call: GPU suite + smoke + acceptance, bench lines (ours: syn20k default,
# syn5k, pmed40; reference arm), p sweep, ncu launch list of the default bench, stamped ncu
# captures of K2 (syn20k) and K2b (syn5k).  Everything lands in gpurun_out/final/.
set -u
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu.txt 2>&1
( time timeout 1500 python -m pytest tests -q -m gpu ) > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 300 ./tests/cpp/_ref/acceptance > $O/acceptance.log 2>&1; echo "acceptance rc=$?" >> $O/acceptance.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ga"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_syn20k.csv $B > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^k_scan$' -c 1 -o $O/k2_scan_syn20k -f python tools/prof_eval.py syn20k scan 2 > $O/ncu_k2.log 2>&1
python tools/ncu_to_json.py $O/k2_scan_syn20k.ncu-rep k_scan syn20k > $O/ncu_k2_json.log 2>&1; cp profiles/ncu_k_scan_syn20k.json $O/
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'^k_gather' -c 1 -o $O/k2b_gather_syn5k -f python tools/prof_eval.py syn5k gather 2 > $O/ncu_k2b.log 2>&1
python tools/ncu_to_json.py $O/k2b_gather_syn5k.ncu-rep k_gather syn5k > $O/ncu_k2b_json.log 2>&1; cp profiles/ncu_k_gather_syn5k.json $O/
timeout 900 python bench.py > $O/bench_syn20k.json 2> $O/bench_syn20k.err
timeout 600 python bench.py --config syn5k --no-ga > $O/bench_syn5k.json 2> $O/bench_syn5k.err
timeout 600 python bench.py --config pmed40 --no-ga > $O/bench_pmed40.json 2> $O/bench_pmed40.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python tools/sweep.py 5 > $O/p_sweep.md 2>&1
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log; head -7 $O/acceptance.log
for f in $O/bench_*.json; do echo "== $f"; head -c 400 $f; echo; done
