#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
for v in default lshdeep1 lshdeep2 default; do
  if [ "$v" = default ]; then lib=paper_2005_11547_b200/libdsk_b200.so; else lib=paper_2005_11547_b200/variants/libdsk_$v.so; fi
  DSK_LIB_PATH=$PWD/$lib timeout 600 python bench_next.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: x=json.loads(l)
    except Exception: continue
    if x['row'].startswith('LshIndex'): print('$v', x['row'], '%.0f'%x['value'], '%.2f ms'%x['ms_per_step'])"
done
