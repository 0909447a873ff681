#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
run() { timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --workload cfg5 $2 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$1 cfg5 $2 dev=%.2f bad=%d'%(d['ms_per_step'],d['status_nonzero']))"; }
for g in 4 6 8 12; do
  DSK_MH_SPLIT_G=$g run "G=$g" "--sets 100000"
  DSK_MH_SPLIT_G=$g run "G=$g" "--sets 2000000"
done
for cl in 8 9 11 12; do
  DSK_MH_SPLIT_CLASS=$cl run "class=$cl" "--sets 100000"
  DSK_MH_SPLIT_CLASS=$cl run "class=$cl" "--sets 2000000"
done
