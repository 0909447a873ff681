export DSK_WL_CACHE=/tmp/wl
for g in 2 3 4 6 8 12; do
  DSK_GMIN=$g timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/s_$g.json 2> gpurun_out/s_$g.err
  python -c "import json;d=json.load(open('gpurun_out/s_$g.json'));print('G>=$g', 'ms=%.2f'%d['ms_per_step'], 'sm=%s'%d['clocks']['sm_mhz'])" || tail -3 gpurun_out/s_$g.err
done
