export DSK_WL_CACHE=/tmp/wl
timeout 600 python -m pytest tests -m gpu -x -q -k "minhash or smoke or host" 2>&1 | tail -1
for spec in "cfg1" "cfg5 --sets 300000"; do
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --workload $spec > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$spec', 'ms=%.3f'%d['ms_per_step'], 'bad=%d'%d['status_nonzero'])"
done
DSK_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu --workload cfg5 --sets 2000000 > gpurun_out/torchrun2.json 2> gpurun_out/torchrun2.err; echo torchrun rc=$?; tail -c 900 gpurun_out/torchrun2.json
DSK_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/torchrun2_ref.json 2> gpurun_out/torchrun2_ref.err; echo torchrun-ref rc=$?; tail -c 300 gpurun_out/torchrun2_ref.json
