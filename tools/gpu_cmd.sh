#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
timeout 1500 python -m pytest tests -q -x -m gpu -k edge 2>&1 | grep -E "Error|error|assert|FAIL|passed|failed|^E " | head -30
