mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_wide_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/r2/t32.log 2>&1; echo rc=$? >> gpurun_out/r2/t32.log
O=gpurun_out/r2/bench32.jsonl; rm -f $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for a in "--config 4 --s 2 --batch 64" "--config 4 --s 1 --batch 32" "--config 1 --s 1"; do
  timeout 300 python bench.py $a $B >> $O 2>> gpurun_out/r2/bench32.err; done
