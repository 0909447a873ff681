#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
for wl in "--workload cfg2" "--workload cfg3 --k 256" "--workload cfg5 --sets 2000000"; do
  for v in default mh1 mh3 mh4 refill4 refill12 threg16 fuse1; do
    if [ "$v" = default ]; then lib=paper_2005_11547_b200/libdsk_b200.so; else lib=paper_2005_11547_b200/variants/libdsk_$v.so; fi
    DSK_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e $wl > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$v FAILED"; continue; }
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', '$wl', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"
  done
done
