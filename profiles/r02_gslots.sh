# large-k minhash: slot arrays in shared memory (teams of 5 for k = 1024) vs global memory (single-warp teams)
export DSK_WL_CACHE=/tmp/wl
for spec in "cfg3 --k 1024" "cfg3 --k 256"; do for g in 0 1; do for rep in 1 2; do
DSK_GLOBAL_SLOTS=$g timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --workload $spec > gpurun_out/ab.json 2> gpurun_out/ab.err || { echo "$spec g=$g failed"; tail -2 gpurun_out/ab.err; continue; }
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$spec global_slots=$g', 'ms=%.2f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"
done; done; done
