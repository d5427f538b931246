#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
python tools/prof_ga.py syn20k 3 device
python tools/prof_ga.py pmed40 3 device
python tools/prof_ga.py syn20k 2 device && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ga_launches.csv python tools/prof_ga.py syn20k 2 device > /dev/null 2>&1
