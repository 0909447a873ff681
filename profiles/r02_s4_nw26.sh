#!/bin/bash
# LSH shard tests; A/B of the 26-warp direct-only LSH first launch (DSK_LSH_NW26=1)
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 900 python -m pytest tests -m gpu -x -q -k "host_multi or rank_shards or lsh_cfg4" > gpurun_out/pytest_shard.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_shard.log
for r in 1 2; do
  bash profiles/ab.sh "--workload cfg4" default | head -1
  DSK_LSH_NW26=1 bash profiles/ab.sh "--workload cfg4" default | head -1 | sed 's/^default/nw26/'
done
DSK_LSH_NW26=1 timeout 600 python -m pytest tests -m gpu -x -q -k "lsh" > gpurun_out/pytest_nw26.log 2>&1; echo pytest-nw26 rc=$?; tail -2 gpurun_out/pytest_nw26.log
