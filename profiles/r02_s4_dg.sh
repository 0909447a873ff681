#!/bin/bash
# direct-only LSH launch: team size 2 (14 teams) vs 1 (28 single-warp teams)
set -u
export DSK_WL_CACHE=/tmp/wl
for r in 1 2; do
  bash profiles/ab.sh "--workload cfg4" default | head -1
  DSK_LSH_DG=1 bash profiles/ab.sh "--workload cfg4" default | head -1 | sed 's/^default/dg1/'
done
DSK_LSH_DG=1 timeout 900 python -m pytest tests -m gpu -x -q -k "lsh or LSH" > gpurun_out/pytest_dg1.log 2>&1; echo pytest-dg1 rc=$?; tail -2 gpurun_out/pytest_dg1.log
