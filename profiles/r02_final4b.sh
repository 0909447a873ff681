#!/bin/bash
# parity report and acceptance shapes on the final build (size split on)
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1200 python profiles/acceptance_shapes.py > gpurun_out/acceptance_shapes.json 2> gpurun_out/acceptance.err; echo acc rc=$?
timeout 2400 python tests/parity_report.py --out gpurun_out/parity_report.json > gpurun_out/parity_report.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/parity_report.log
