#!/bin/bash
# compile-time knobs re-measured on the 28-warp kernels (one round each; winners get a second look)
set -u
export DSK_WL_CACHE=/tmp/wl
for wl in "--workload cfg4" "--workload cfg3 --k 256"; do
  for v in default opq0 opq2 opqtb0 selni ptsm seek0 nofuse sel32_0 thhit16 tharea16; do
    if [ "$v" = default ]; then lib=paper_2005_11547_b200/libdsk_b200.so; else lib=paper_2005_11547_b200/variants/libdsk_$v.so; fi
    DSK_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e $wl > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$v FAILED"; continue; }
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', '$wl', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"
  done
done
