#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "table or ordering or parity or instance or baseline_sizes or tables_and_every" > gpurun_out/k1_pytest.log 2>&1; tail -2 gpurun_out/k1_pytest.log
for n in 20000 10000 5000 900; do
  python tools/time_k1.py $n; PMB_K1_PREP=0 python tools/time_k1.py $n
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_(build_rows|prep|validate|transpose_costs)' python tools/prof_eval.py syn20k scan 1 > gpurun_out/k1_ncu.log 2>&1; grep -E "k_build|k_prep|duration|dram__" gpurun_out/k1_ncu.log | head -16
ncu --set full --import-source on --clock-control none -k regex:'^k_build_rows_cs' -c 1 -o gpurun_out/k1_cs_syn20k -f python tools/prof_eval.py syn20k scan 1 > /dev/null 2>&1; ls -la gpurun_out/k1_cs_syn20k.ncu-rep
