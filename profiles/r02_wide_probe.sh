# Does the wide (teams of 2) shape still win anywhere for minhash?  uniform large sets, small k
export DSK_WL_CACHE=/tmp/wl
for spec in "cfg2 --k 128" "cfg2 --k 64" "cfg4 --k 128"; do for v in default 20 22; do
if [ $v = default ]; then E=""; else E="DSK_NW=$v"; fi
env $E timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --workload $spec > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$spec $v failed"; tail -2 gpurun_out/ab.err; continue; }
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$spec NW=$v', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"
done; done
