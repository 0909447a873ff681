#!/bin/bash
# size split of single-warp-team minhash launches (DSK_MH_SPLIT=1): correctness, cfg5 device-resident and e2e at small chunks
set -u
export DSK_WL_CACHE=/tmp/wl
DSK_MH_SPLIT=1 timeout 600 python profiles/soak.py 24 7 2>&1 | grep -v "same=True oracle_ok=True" | tail -3
DSK_MH_SPLIT=1 timeout 900 python -m pytest tests -m gpu -x -q -k "cfg5 or zipf or skew or full_size or large or shard" > gpurun_out/pytest_split.log 2>&1; echo pytest-split rc=$?; tail -2 gpurun_out/pytest_split.log
for v in 0 1; do
  DSK_MH_SPLIT=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --workload cfg5 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('split=$v cfg5 full dev=%.2f bad=%d launches=%d'%(d['ms_per_step'],d['status_nonzero'],d['gpu_launches']))"
  DSK_MH_SPLIT=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --workload cfg5 --sets 100000 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('split=$v cfg5 1e5 dev=%.2f bad=%d'%(d['ms_per_step'],d['status_nonzero']))"
  for mb in 32 128 512; do
    echo "split=$v chunk=$mb"; DSK_MH_SPLIT=$v DSK_CHUNK_MB=$mb DSK_LIB_PATH=$PWD/paper_2005_11547_b200/libdsk_b200.so timeout 900 python profiles/e2e_probe.py cfg5 2000000 3 2>&1 | tail -2 | head -1
  done
done
