# cfg5 team shape vs batch size: default rule (24 warps x teams of 2) vs 20 single-warp teams
export DSK_WL_CACHE=/tmp/wl
for n in 300000 1000000 10000000; do for v in default 20; do
if [ $v = default ]; then E=""; else E="DSK_NW=$v"; fi
env $E timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --workload cfg5 --sets $n > gpurun_out/ab.json 2> gpurun_out/ab.err || { tail -3 gpurun_out/ab.err; continue; }
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('cfg5 n=$n NW=$v', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"
done; done
