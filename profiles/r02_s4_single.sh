#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
for r in 1 2; do
  bash profiles/ab.sh "--workload cfg4" default | head -1
  DSK_LSH_SINGLE=0 bash profiles/ab.sh "--workload cfg4" default | head -1 | sed 's/^default/runtimeG/'
done
