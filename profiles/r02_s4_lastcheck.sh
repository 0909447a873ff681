#!/bin/bash
# final HEAD: GPU suite, smoke, then the suite under the DSK_DEBUG build (+ direct-first forced), soak
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
DSK_LIB_PATH=$PWD/paper_2005_11547_b200/variants/libdsk_debug.so timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_debug.log 2>&1; echo pytest-debug rc=$?; tail -2 gpurun_out/pytest_debug.log
DSK_LIB_PATH=$PWD/paper_2005_11547_b200/variants/libdsk_debug.so DSK_MH_DIRECT=1 timeout 2400 python -m pytest tests -m gpu -x -q -k "not lsh" > gpurun_out/pytest_debug_direct.log 2>&1; echo pytest-debug-direct rc=$?; tail -2 gpurun_out/pytest_debug_direct.log
DSK_LIB_PATH=$PWD/paper_2005_11547_b200/variants/libdsk_debug.so timeout 900 python profiles/soak.py 20 21 2>&1 | tail -1
