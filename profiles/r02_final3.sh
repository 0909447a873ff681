#!/bin/bash
# Round-2 evidence pass on the final build (session 4: 28-warp direct-only LSH
# launch, direct-first minhash): GPU suite, smoke, default bench (cfg4, e2e +
# CPU baselines), reference arm, per-workload device timings, launch list,
# ncu --set full captures, acceptance shapes, parity report over the SURVEY
# 8(d) subsets.  Outputs under gpurun_out/.
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref rc=$?
bash profiles/quick_all.sh 2>&1 | head -7 > gpurun_out/quick_all.txt; cat gpurun_out/quick_all.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc=$?
SKIP=6 bash profiles/ncu_capture.sh r02f_lsh_cfg4 lsh_kernel --workload cfg4 --sets 200000
SKIP=3 bash profiles/ncu_capture.sh r02f_mh_cfg2 minhash_kernel --workload cfg2
timeout 1200 python profiles/acceptance_shapes.py > gpurun_out/acceptance_shapes.json 2> gpurun_out/acceptance.err; echo acc rc=$?
timeout 2400 python tests/parity_report.py --out gpurun_out/parity_report.json > gpurun_out/parity_report.log 2>&1; echo parity rc=$?; tail -9 gpurun_out/parity_report.log
