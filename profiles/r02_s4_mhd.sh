#!/bin/bash
# direct-first minhash (DSK_MH_DIRECT=1: direct-only engine on 28/24 warps, general launch for the rest) vs default
set -u
export DSK_WL_CACHE=/tmp/wl
for spec in "cfg3 --k 64" "cfg3 --k 256" "cfg3 --k 1024" "cfg5" "cfg2"; do
  for v in 0 1; do
    DSK_MH_DIRECT=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --workload $spec > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$spec $v FAILED"; tail -3 gpurun_out/ab.err; continue; }
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('direct=$v', '$spec', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'], 'launches=%d'%d['gpu_launches'], 'phi=%s'%d['phi_hist'])"
  done
done
DSK_MH_DIRECT=1 timeout 1500 python -m pytest tests -m gpu -x -q -k "not lsh" > gpurun_out/pytest_mhd.log 2>&1; echo pytest-direct rc=$?; tail -3 gpurun_out/pytest_mhd.log
