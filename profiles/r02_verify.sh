#!/bin/bash
# round-2 re-entry check: GPU tests, smoke, default bench, per-workload quick numbers
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?; cat gpurun_out/bench_default.json | head -c 3000
bash profiles/quick_all.sh 2>&1 | head -12
