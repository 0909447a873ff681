#!/bin/bash
# last evidence refresh of the round (after the host chunk sizes and the size split):
# default bench + reference arm, per-workload timings, launch list, cfg5 capture (both launches of the size split)
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref rc=$?
bash profiles/quick_all.sh 2>&1 | head -7 > gpurun_out/quick_all.txt; cat gpurun_out/quick_all.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc=$?
SKIP=6 COUNT=2 bash profiles/ncu_capture.sh r02f_mh_cfg5 minhash_kernel --workload cfg5 --sets 1000000
timeout 900 python bench_next.py > gpurun_out/bench_next.jsonl 2> gpurun_out/bench_next.err; echo bench_next rc=$?; tail -5 gpurun_out/bench_next.jsonl | cut -c1-300
