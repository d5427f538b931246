#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "parity or smoke" 2>&1 | tail -1
for p in 10 20 50 100 200 500 1000; do
python tools/time_eval.py sweep:$p gather 5 "auto" 1
python tools/time_eval.py sweep:$p scan 5 "auto" 1
done
python tools/time_eval.py syn5k gather 10 "auto" 1
python tools/time_eval.py syn5k scan 10 "auto 32,16" 1
python tools/time_eval.py syn20k gather 3 "auto" 1
python tools/time_eval.py syn20k scan 10 "auto 32,16" 1
python tools/time_eval.py pmed40 gather 10 "auto" 1
