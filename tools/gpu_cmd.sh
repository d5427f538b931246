#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "ga or island or ingest" 2>&1 | tail -1
python tools/prof_ga.py pmed40 1 reference > /dev/null; python tools/prof_ga.py pmed40 5 reference; python tools/prof_ga.py pmed40 5 device
