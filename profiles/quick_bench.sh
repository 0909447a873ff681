#!/bin/bash
# quick per-workload timings (device-resident, no e2e/cpu legs); one line each
for spec in "cfg2" "cfg3 --k 64" "cfg3 --k 256" "cfg3 --k 1024" "cfg4" "cfg5 --sets 1000000" "cfg1"; do
  set -- $spec
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --workload $spec > gpurun_out/qb.json 2> gpurun_out/qb.err || { echo "$spec FAILED"; tail -3 gpurun_out/qb.err; continue; }
  python -c "import json;d=json.load(open('gpurun_out/qb.json'));print('$spec', 'ms=%.2f'%d['ms_per_step'], 'sets/s=%.3g'%d['value'], 'darts/s=%.3g'%d['darts_per_sec'], 'alu_frac=%.3f'%d['roofline']['frac'], 'sm=%s'%d['clocks']['sm_mhz'], 'bad=%d'%d['status_nonzero'], 'phi=%s'%d['phi_hist'])"
done
