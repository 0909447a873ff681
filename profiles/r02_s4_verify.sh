#!/bin/bash
# Session-4 check of HEAD (walker seek table build): GPU suite, smoke, default
# bench, per-workload device timings, ncu --set full of the cfg4 LSH kernel.
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
bash profiles/quick_all.sh 2>&1 | head -7 > gpurun_out/quick_all.txt; cat gpurun_out/quick_all.txt
SKIP=6 bash profiles/ncu_capture.sh r02s4_lsh_cfg4 lsh_kernel --workload cfg4 --sets 200000
SKIP=3 bash profiles/ncu_capture.sh r02s4_mh_cfg2 minhash_kernel --workload cfg2
