#!/bin/bash
# (historical: the window tie pass was measured slower and removed -- DESIGN.md §4 K1; PMB_K1_WIN no longer exists)
# K1 counting sort: window tie pass (default) vs the thread-per-bucket sort (PMB_K1_WIN=0):
# table parity, set_instance wall times, and the kernel's ncu duration at syn20k.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "table or ordering or parity or instance or baseline or tail" > gpurun_out/k1_win_pytest.log 2>&1; tail -2 gpurun_out/k1_win_pytest.log
for r in 1 2; do for n in 20000 10000 5000 900; do for w in 1 0; do
  echo "win=$w $(PMB_K1_WIN=$w python tools/time_k1.py $n)"
done; done; done
for w in 1 0; do
  PMB_K1_WIN=$w ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_build_rows_cs' -c 1 python tools/prof_eval.py syn20k scan 1 > gpurun_out/k1_win_ncu_$w.log 2>&1
  echo "win=$w"; grep -E "duration|inst_executed|dram__" gpurun_out/k1_win_ncu_$w.log | head -4
done
