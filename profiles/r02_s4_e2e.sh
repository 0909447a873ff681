#!/bin/bash
# cfg4 end-to-end (dsk_lsh_csr_host, pinned): chunk size / ramp alternatives
set -u
export DSK_WL_CACHE=/tmp/wl
run() { timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$1', 'dev=%.2f e2e=%.2f pageable=%.2f'%(d['ms_per_step'],d['e2e']['ms_per_step'],d['e2e_pageable']['ms_per_step']))"; }
run default
DSK_CHUNK_MB=128 run chunk128
DSK_CHUNK_MB=32 run chunk32
DSK_RAMP_MB=32,8 run ramp32_8
DSK_RAMP_MB=8,4 run ramp8_4
DSK_RAMP_MB=16,16 run ramp16_16
run default
