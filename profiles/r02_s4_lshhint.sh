#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 900 python -m pytest tests -m gpu -x -q -k "lsh or LSH or integration or abi or symbol" > gpurun_out/pytest_lsh.log 2>&1; echo pytest-lsh rc=$?; tail -2 gpurun_out/pytest_lsh.log
for n in 30000 300000; do timeout 300 python profiles/lsh_skew_probe.py $n 2>&1 | tail -1; done
bash profiles/quick_all.sh 2>&1 | head -1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --workload cfg4 --sets 125000 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg4 125k sets: dev=%.2f e2e=%.2f'%(d['ms_per_step'],d['e2e']['ms_per_step']))"
