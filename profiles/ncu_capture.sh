#!/bin/bash
# ncu --set full capture (source-attributed) of one sketch kernel launch of
# a bench workload: profiles/ncu_capture.sh <name> <kernel-regex> <bench args...>
# The bench command runs once WITHOUT ncu first (must exit 0), then under ncu
# skipping the warm-up launches (SKIP, default 3: one sketch launch per
# warm-up step; LSH launches twice per step -> SKIP=6).  Output:
# gpurun_out/<name>.ncu-rep
NAME=$1; KREG=$2; shift 2
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu $*"
timeout 900 $CMD > gpurun_out/${NAME}_plain.json 2> gpurun_out/${NAME}_plain.err || { echo "plain run failed"; exit 1; }
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:$KREG -s ${SKIP:-3} -c ${COUNT:-1} \
  -o gpurun_out/$NAME -f $CMD > gpurun_out/${NAME}_ncu.log 2>&1
echo "ncu $NAME rc=$?"
