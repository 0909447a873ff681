#!/bin/bash
# A/B timing of library variants over several workloads (2 rounds each):
#   bash profiles/ab_multi.sh "<variant> <variant> ..." "cfg4" "cfg2" "cfg3 --k 256" ...
VARS=$1; shift
for wl in "$@"; do bash profiles/ab.sh "--workload $wl" $VARS; done
