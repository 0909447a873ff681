#!/bin/bash
# A/B timing of library variants on one workload (device-resident, 5 steps):
#   bash profiles/ab.sh "<bench args>" default old ssel0 ...
# "default" = paper_2005_11547_b200/libdsk_b200.so, else variants/libdsk_<name>.so
ARGS=$1; shift
export DSK_WL_CACHE=/tmp/wl
for v in "$@" "$@"; do
  if [ "$v" = default ]; then lib=paper_2005_11547_b200/libdsk_b200.so; else lib=paper_2005_11547_b200/variants/libdsk_$v.so; fi
  DSK_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e $ARGS > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$v FAILED"; tail -3 gpurun_out/ab.err; continue; }
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', '$ARGS', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'], 'sm=%s'%d['clocks']['sm_mhz'])"
done
