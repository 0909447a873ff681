#!/bin/bash
# second part of the final evidence pass (gpurun_out/ is limited to 64 MiB per call)
set -u
export DSK_WL_CACHE=/tmp/wl
SKIP=6 bash profiles/ncu_capture.sh r02f_mh_cfg3_k1024 minhash_kernel --workload cfg3 --k 1024 --sets 200000
SKIP=3 bash profiles/ncu_capture.sh r02f_mh_cfg5 minhash_kernel --workload cfg5 --sets 1000000
