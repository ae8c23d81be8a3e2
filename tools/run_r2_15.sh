mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_wide_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/r2/t16.log 2>&1; echo rc=$? >> gpurun_out/r2/t15.log
O=gpurun_out/r2/bench16.jsonl; rm -f $O
B="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for a in "--config 4 --s 1 --batch 32" "--config 1 --s 1" "--config 0"; do
  timeout 300 python bench.py $a $B >> $O 2>> gpurun_out/r2/bench16.err
  FGF_DEV=1 FGF_ENGINE=notiny timeout 300 python bench.py $a $B >> $O 2>> gpurun_out/r2/bench16.err
done
