#!/bin/bash
# direct-only LSH first launch: CTA width 24 / 26 / 28 warps (DSK_LSH_DNW), then the LSH tests at the default
set -u
export DSK_WL_CACHE=/tmp/wl
for r in 1 2; do
  for w in 28 32; do
    DSK_LSH_DNW=$w bash profiles/ab.sh "--workload cfg4" default | head -1 | sed "s/^default/dnw$w/"
  done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "lsh or LSH" > gpurun_out/pytest_dnw.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_dnw.log
