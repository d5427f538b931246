#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
python tools/time_eval.py syn5k scan 10 "auto 64,12 64,10 64,8" 1
python tools/time_eval.py sweep:100 scan 10 "auto 64,10 64,8 64,6" 1
python tools/time_eval.py sweep:200 scan 10 "auto 64,10 64,8" 1
python tools/time_eval.py pmed40 scan 10 "auto 64,16 64,12" 1
