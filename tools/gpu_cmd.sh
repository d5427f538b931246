#!/bin/bash
mkdir -p gpurun_out
exec > gpurun_out/timing.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "cli" 2>&1 | grep -E "Error|error|assert|FAIL|passed|failed|^E " | head -30
