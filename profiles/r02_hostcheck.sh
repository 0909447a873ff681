export DSK_WL_CACHE=/tmp/wl
timeout 900 python -m pytest tests -m gpu -x -q -k "host or multi or pageable or abi or stub" 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/b4.json 2> gpurun_out/b4.err
python -c "import json;d=json.load(open('gpurun_out/b4.json'));print('cfg4', 'ms=%.2f'%d['ms_per_step'], 'e2e', round(d['e2e']['ms_per_step'],1), 'pageable', round(d['e2e_pageable']['ms_per_step'],1))"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --workload cfg2 > gpurun_out/b2.json 2> gpurun_out/b2.err
python -c "import json;d=json.load(open('gpurun_out/b2.json'));print('cfg2', 'ms=%.2f'%d['ms_per_step'], 'e2e', round(d['e2e']['ms_per_step'],1), 'pageable', round(d['e2e_pageable']['ms_per_step'],1))"
