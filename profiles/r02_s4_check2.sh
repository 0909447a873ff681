#!/bin/bash
# full GPU suite + per-workload timings with the direct-first hints in effect + host-path e2e of cfg3
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
bash profiles/quick_all.sh 2>&1 | head -7 > gpurun_out/quick_all.txt; cat gpurun_out/quick_all.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --workload cfg3 --k 256 > gpurun_out/cfg3_e2e.json 2> gpurun_out/cfg3_e2e.err; python -c "
import json;d=json.load(open('gpurun_out/cfg3_e2e.json'));print('cfg3 k256 dev ms=%.2f e2e ms=%.2f pageable ms=%.2f launches=%d'%(d['ms_per_step'],d['e2e']['ms_per_step'],d['e2e_pageable']['ms_per_step'],d['gpu_launches']))"
