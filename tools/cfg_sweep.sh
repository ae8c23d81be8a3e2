#!/bin/bash
# Development sweep over BASELINE.json configs / s values (bench.py lines, no e2e / cpu).
for a in "$@"; do
  python bench.py $a --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cfg.log 2>&1 || { echo "$a FAILED"; tail -3 gpurun_out/cfg.log; continue; }
  python -c "import json;d=json.loads(open('gpurun_out/cfg.log').read().strip().splitlines()[-1]);print('$a', round(d['value']), 'Mpx/s', round(d['ms_per_step'],3), 'ms', d.get('hbm_whole_filter',{}).get('model_GBs'), {k:(round(v['ms_per_launch'],3), v['launches_per_step']) for k,v in d.get('kernels',{}).items() if v['launches_per_step']})"
done
