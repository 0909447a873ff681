#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$1', 'dev=%.2f e2e=%.2f pageable=%.2f'%(d['ms_per_step'],d['e2e']['ms_per_step'],d['e2e_pageable']['ms_per_step']))"; }
DSK_CHUNK_MB=128 run chunk128
DSK_CHUNK_MB=256 run chunk256
DSK_CHUNK_MB=192 run chunk192
DSK_CHUNK_MB=128 DSK_RAMP_MB=32,8 run chunk128_ramp32
