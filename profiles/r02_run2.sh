free -g; nproc; nvidia-smi -L
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_cfg4.json 2> gpurun_out/r2_cfg4.err; echo cfg4 rc=$?
timeout 1200 python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_cfg5.json 2> gpurun_out/r2_cfg5.err; echo cfg5 rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
