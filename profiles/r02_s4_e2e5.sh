#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
for mb in 64 256 512 1024 4096; do
  echo "chunk $mb"; DSK_CHUNK_MB=$mb DSK_LIB_PATH=$PWD/paper_2005_11547_b200/libdsk_b200.so timeout 900 python profiles/e2e_probe.py cfg5 2000000 3 2>&1 | tail -2
done
