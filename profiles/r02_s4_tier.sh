#!/bin/bash
# two-tier LSH hit buffer: LSH test subset, then A/B against the HEAD build
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1500 python -m pytest tests -m gpu -x -q -k "lsh or LSH" > gpurun_out/pytest_lsh.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_lsh.log
bash profiles/ab.sh "--workload cfg4" default head
for f in 0.6 0.65 0.8; do
  echo "tier $f"; DSK_LSH_TIER=$f bash profiles/ab.sh "--workload cfg4" default | head -1
done
