#!/bin/bash
# device-resident timings of every workload (no e2e / CPU legs), one line each
export DSK_WL_CACHE=${DSK_WL_CACHE:-/tmp/wl}
for spec in "cfg4" "cfg2" "cfg3 --k 64" "cfg3 --k 256" "cfg3 --k 1024" "cfg5" "cfg1"; do
  set -- $spec
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --workload $spec > gpurun_out/qa.json 2> gpurun_out/qa.err || { echo "$spec FAILED"; tail -3 gpurun_out/qa.err; continue; }
  python -c "import json;d=json.load(open('gpurun_out/qa.json'));r=d['roofline'] or {};print('$spec', 'ms=%.2f'%d['ms_per_step'], 'sets/s=%.4g'%d['value'], 'darts/s=%.4g'%d['darts_per_sec'], 'useful=%.3f'%d['roofline_useful']['frac'], 'issue=%s'%r.get('frac'), 'sm=%s'%d['clocks']['sm_mhz'], 'bad=%d'%d['status_nonzero'], 'phi=%s'%d['phi_hist'])"
done
