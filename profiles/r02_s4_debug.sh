#!/bin/bash
# GPU suite under the DSK_DEBUG build (ring-capacity / cursor / slot-index assertions in the engine),
# incl. the packed-queue 28-warp kernels; then timings of the wide_g = 3 rule
set -u
export DSK_WL_CACHE=/tmp/wl
DSK_LIB_PATH=$PWD/paper_2005_11547_b200/variants/libdsk_debug.so timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_debug.log 2>&1; echo pytest-debug rc=$?; tail -2 gpurun_out/pytest_debug.log
DSK_LIB_PATH=$PWD/paper_2005_11547_b200/variants/libdsk_debug.so DSK_MH_DIRECT=1 timeout 2400 python -m pytest tests -m gpu -x -q -k "not lsh" > gpurun_out/pytest_debug_direct.log 2>&1; echo pytest-debug-direct rc=$?; tail -2 gpurun_out/pytest_debug_direct.log
bash profiles/quick_all.sh 2>&1 | head -3; 
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --workload cfg2 --k 64 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg2 k64 ms=%.2f'%d['ms_per_step'])"
DSK_NW=22 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --workload cfg2 --k 64 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg2 k64 nw22 ms=%.2f'%d['ms_per_step'])"
