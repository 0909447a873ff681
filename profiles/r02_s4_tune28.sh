#!/bin/bash
# 28 x 1 direct-only LSH launch (default now): LSH tests, walker run / refill variants
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 900 python -m pytest tests -m gpu -x -q -k "lsh or LSH" > gpurun_out/pytest_lsh.log 2>&1; echo pytest-lsh rc=$?; tail -2 gpurun_out/pytest_lsh.log
bash profiles/ab.sh "--workload cfg4" default run2 run4 refill4 refill12
