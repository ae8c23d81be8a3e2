#!/bin/bash
# e2e (fgf_filter_host_ex, config 4, 256 images) against the pipeline slot size.
for mb in 64 128 256 512 1024 2048; do
  FGF_DEV=1 FGF_HOST_CHUNK_MB=$mb python bench.py --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 4 2>/dev/null | python -c "
import sys, json
j = json.loads(sys.stdin.read()); print('chunk MB', sys.argv[1], 'e2e', round(j['e2e']['value']), 'Mpixel/s')" $mb
done
