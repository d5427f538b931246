#!/bin/bash
# K1 (set_instance) after the fused prep pass: parity tests, wall times (prep on/off), launch list.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu -k "table or ordering or parity or ingest or instance or baseline" > gpurun_out/k1_pytest.log 2>&1; tail -2 gpurun_out/k1_pytest.log
for n in 20000 10000 5000 900; do
  python tools/time_k1.py $n; PMB_K1_PREP=0 python tools/time_k1.py $n
done
python tools/prof_eval.py syn20k scan 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_(build_rows|prep|validate|transpose_costs)' python tools/prof_eval.py syn20k scan 1 > gpurun_out/k1_ncu.log 2>&1; grep -E "k_build|k_prep|k_valid|k_transp|duration|dram__" gpurun_out/k1_ncu.log | head -24
PMB_K1_PREP=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_(build_rows|prep|validate|transpose_costs)' python tools/prof_eval.py syn20k scan 1 > gpurun_out/k1_ncu_old.log 2>&1; grep -E "k_build|k_prep|k_valid|k_transp|duration|dram__" gpurun_out/k1_ncu_old.log | head -24
