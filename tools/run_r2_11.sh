mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_lowres_fused_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/r2/k13_12.log 2>&1; echo rc=$? >> gpurun_out/r2/k13_11.log
O=gpurun_out/r2/bench12.jsonl; rm -f $O
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O 2>> gpurun_out/r2/bench12.err; done
