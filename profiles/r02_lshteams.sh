export DSK_WL_CACHE=/tmp/wl
for g in 2 3 4; do for rep in 1 2; do
DSK_GMIN=$g timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --workload cfg4 > gpurun_out/ab.json 2> gpurun_out/ab.err || { tail -2 gpurun_out/ab.err; continue; }
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('cfg4 GMIN=$g', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"
done; done
