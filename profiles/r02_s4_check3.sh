#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
bash profiles/quick_all.sh 2>&1 | head -7 > gpurun_out/quick_all.txt; cat gpurun_out/quick_all.txt
