#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "parity or smoke" 2>&1 | tail -1
python tools/time_eval.py syn20k scan 10 "auto 32,14 32,12 32,10" 1
python tools/time_eval.py syn5k scan 10 "auto 32,14" 1
python tools/time_eval.py sweep:100 scan 10 "auto" 1
python tools/time_eval.py pmed40 scan 10 "auto" 1
