#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
for lib in paper_2005_11547_b200/variants/libdsk_old.so paper_2005_11547_b200/libdsk_b200.so; do
  DSK_LIB_PATH=$PWD/$lib timeout 900 python profiles/e2e_probe.py cfg5 2000000 3 2>&1 | tail -2
done
nproc; free -g | head -2
