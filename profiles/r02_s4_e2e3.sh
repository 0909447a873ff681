#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
run() { timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu $WL > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$1', '$WL', 'dev=%.2f e2e=%.2f pageable=%.2f'%(d['ms_per_step'],d['e2e']['ms_per_step'],d['e2e_pageable']['ms_per_step']))"; }
for WL in "--workload cfg3 --k 256" "--workload cfg3 --k 64" "--workload cfg2" "--workload cfg5 --sets 2000000"; do
  DSK_CHUNK_MB=16 run chunk16
  DSK_CHUNK_MB=24 run chunk24
  DSK_CHUNK_MB=32 run chunk32
  DSK_CHUNK_MB=48 run chunk48
done
