#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "parity or smoke or edge" 2>&1 | tail -1
python tools/time_eval.py syn20k scan 10 "auto 32,16 32,14" 1
python tools/time_eval.py syn5k scan 10 "auto" 1
python tools/time_eval.py sweep:200 scan 10 "auto" 1
python tools/time_eval.py sweep:1000 scan 10 "auto" 1
python tools/time_eval.py pmed40 scan 10 "auto" 1
