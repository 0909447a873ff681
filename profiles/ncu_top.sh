#!/bin/bash
# ncu full capture of the minhash kernel on the default bench workload (cfg2)
ARGS="${@:-}"
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu $ARGS"
timeout 300 $CMD > gpurun_out/b_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:minhash_kernel -s 3 -c 1 -o gpurun_out/prof_cur -f $CMD > gpurun_out/ncu_full.log 2>&1
echo ncu=$?
