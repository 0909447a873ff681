#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for s in 11 12; do timeout 500 python profiles/soak.py 30 $s 2>&1 | grep -v "same=True oracle_ok=True" | tail -2; done
bash profiles/quick_all.sh 2>&1 | head -7 > gpurun_out/quick_all.txt; cat gpurun_out/quick_all.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --workload cfg5 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('cfg5 dev=%.2f e2e=%.2f pageable=%.2f'%(d['ms_per_step'],d['e2e']['ms_per_step'],d['e2e_pageable']['ms_per_step']))"
