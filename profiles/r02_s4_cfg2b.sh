#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
for r in 1 2; do
  bash profiles/ab.sh "--workload cfg2" default | head -1
  DSK_NW=22 bash profiles/ab.sh "--workload cfg2" default | head -1 | sed 's/^default/nw22/'
  DSK_NW=20 bash profiles/ab.sh "--workload cfg2" default | head -1 | sed 's/^default/nw20/'
done
