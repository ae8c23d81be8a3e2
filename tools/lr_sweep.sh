#!/bin/bash
# Development sweep of the fused low-res kernel's geometry knobs (FGF_LR_*), config 4 s=4.
for cfg in "$@"; do
  env $cfg python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sweep.log 2>&1 || { echo "$cfg FAILED"; tail -3 gpurun_out/sweep.log; continue; }
  python -c "import json,sys;d=json.loads(open('gpurun_out/sweep.log').read().strip().splitlines()[-1]);print('$cfg', round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items() if v['launches_per_step']})"
done
