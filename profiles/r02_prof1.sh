#!/bin/bash
# round-2 source-attributed captures of the current build (cfg4 LSH 2e5 sets, cfg2 minhash)
SKIP=6 bash profiles/ncu_capture.sh r02_lsh_cfg4 lsh_kernel --workload cfg4 --sets 200000
SKIP=3 bash profiles/ncu_capture.sh r02_mh_cfg2 minhash_kernel --workload cfg2
ls -la gpurun_out/*.ncu-rep
