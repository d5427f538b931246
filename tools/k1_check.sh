#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "${PYTEST_K:-table or ordering or parity or ingest or instance}" > gpurun_out/k1_pytest.log 2>&1; tail -2 gpurun_out/k1_pytest.log
for n in 20000 5000 900; do
  python tools/time_k1.py $n; PMB_K1=radix python tools/time_k1.py $n
done
python tools/prof_eval.py syn20k scan 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_build_rows' python tools/prof_eval.py syn20k scan 1 2>&1 | grep -E "k_build|duration|dram__" | head -12
