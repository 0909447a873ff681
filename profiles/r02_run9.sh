timeout 1200 python -m pytest tests -m gpu -x -q -k "lsh or LshIndex or smoke or cli" > gpurun_out/pytest_lsh.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_lsh.log
export DSK_WL_CACHE=/tmp/wl
for c in 1 0; do
DSK_LSH_COMPACT=$c timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b4c$c.json 2>gpurun_out/b4c$c.err
python -c "import json;d=json.load(open('gpurun_out/b4c$c.json'));print('cfg4 compact=$c', 'ms=%.2f'%d['ms_per_step'], 'useful=%.3f'%d['roofline_useful']['frac'], d['phi_hist'], 'bad', d['status_nonzero'], 'launches', d['gpu_launches'])" || tail -3 gpurun_out/b4c$c.err
done
SKIP=6 bash profiles/ncu_capture.sh r02_lsh_cfg4e lsh_kernel --workload cfg4 --sets 200000
python profiles/summ.py gpurun_out/r02_lsh_cfg4e.ncu-rep | grep "dram\|duration\|inst_executed.sum\|stalls"
