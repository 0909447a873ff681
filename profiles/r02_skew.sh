export DSK_WL_CACHE=/tmp/wl
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu --workload cfg5 > gpurun_out/b5.json 2> gpurun_out/b5.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/b5.json'));print('cfg5', 'ms=%.2f'%d['ms_per_step'], 'e2e', d['e2e'], 'bad=%d'%d['status_nonzero'])"
for spec in "cfg2" "cfg2 --k 128" "cfg3 --k 64"; do
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --workload $spec > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$spec', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"
done
