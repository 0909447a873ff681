#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1200 python -m pytest tests -m gpu -x -q -k "host or abi or pinned or pageable or multi or concurrent or integration" > gpurun_out/pytest_host.log 2>&1; echo pytest-host rc=$?; tail -2 gpurun_out/pytest_host.log
run() { timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu $WL > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$WL', 'dev=%.2f e2e=%.2f pageable=%.2f'%(d['ms_per_step'],d['e2e']['ms_per_step'],d['e2e_pageable']['ms_per_step']))"; }
for WL in "--workload cfg2" "--workload cfg3 --k 64" "--workload cfg3 --k 256" "--workload cfg5"; do run; done
