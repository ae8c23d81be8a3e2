#!/bin/bash
# Single-frame row-band host pipeline: parity, then config 1 e2e with and without it.
FGF_FUZZ_HOST_SEEDS=600 timeout 900 python -m pytest tests/test_fuzz_gpu.py tests/test_parity_gpu.py -x -q -k "host" 2>&1 | tail -6
for rep in 1 2; do for nb in "" "FGF_HOST_NOBANDS=1"; do
  env FGF_DEV=1 $nb python bench.py --config 1 --no-cpu-baseline --steps 20 --warmup 3 --e2e-steps 50 2>/dev/null | python -c "
import sys, json
j = json.loads(sys.stdin.read()); e = j['e2e']; print(sys.argv[1] or 'bands', 'e2e', round(e['value']), 'Mpixel/s =', round(8.2944 / e['value'] * 1e3, 3), 'ms per frame')" "$nb"
done; done
