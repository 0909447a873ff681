export DSK_WL_CACHE=/tmp/wl
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
bash profiles/ab_multi.sh "head default" "cfg2" "cfg1"
bash profiles/ab_multi.sh "head ch128" "cfg4"
for nw in 24 22 20; do for rep in 1 2; do
DSK_NW=$nw timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --workload cfg5 --sets 2000000 > gpurun_out/ab.json 2> gpurun_out/ab.err || { tail -3 gpurun_out/ab.err; continue; }
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('cfg5 2e6 NW=$nw', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"
done; done
for rep in 1 2; do timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --workload cfg5 --sets 2000000 > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('cfg5 2e6 default', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"; done
