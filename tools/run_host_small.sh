#!/bin/bash
# Small batches through fgf_filter_host_ex: >= 4 chunks (default) against one 256 MB slot.
timeout 900 python -m pytest tests/test_fuzz_gpu.py tests/test_parity_gpu.py -x -q -k "host" 2>&1 | tail -3
for rep in 1 2; do for a in "--config 1 --batch 8|" "--config 1 --batch 8|FGF_HOST_CHUNK_MB=256" "--config 0 --batch 64|" "--config 0 --batch 64|FGF_HOST_CHUNK_MB=256" "--config 3 --batch 6|" "--config 3 --batch 6|FGF_HOST_CHUNK_MB=256"; do
  args=${a%%|*}; envs=${a##*|}
  env FGF_DEV=1 $envs python bench.py $args --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 30 2>/dev/null | python -c "
import sys, json
j = json.loads(sys.stdin.read()); e = j['e2e']; print(sys.argv[1], '|', sys.argv[2] or 'default', '| e2e', round(e['value']), 'Mpixel/s')" "$args" "$envs"
done; done
