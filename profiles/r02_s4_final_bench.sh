#!/bin/bash
set -u
export DSK_WL_CACHE=/tmp/wl
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?; python -c "
import json;d=json.load(open('gpurun_out/bench_default.json'));print('cfg4 value=%.4g ms=%.2f e2e=%.4g roofline=%.3f launches=%d steps=%d'%(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['gpu_launches'],d['steps']))"
DSK_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --sets 200000 --no-cpu > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo torchrun rc=$?; tail -1 gpurun_out/bench_2rank.json | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('2 ranks (gloo, one GPU: code path only): n_gpus=%d sets=%d value=%.4g scaling=%s'%(d['n_gpus'],d['config']['sets'],d['value'],d['scaling']))"
DSK_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_2rank_ref.json 2> gpurun_out/bench_2rank_ref.err; echo torchrun-ref rc=$?; tail -1 gpurun_out/bench_2rank_ref.json | cut -c1-200
