#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
bash profiles/ab.sh "--workload cfg4" default fzhi
bash profiles/ab.sh "--workload cfg3 --k 256" default fzhi | head -2
bash profiles/ab.sh "--workload cfg2" default fzhi | head -2
