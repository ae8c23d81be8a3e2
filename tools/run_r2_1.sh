mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_wide_gpu.py -x -q > gpurun_out/r2/wide1.log 2>&1; echo rc=$? >> gpurun_out/r2/wide1.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/gputest1.log 2>&1; echo rc=$? >> gpurun_out/r2/gputest1.log
for a in "--config 4 --s 1 --batch 32" "--config 1 --s 1" "--config 4 --s 2 --batch 64" "--config 4"; do
  timeout 300 python bench.py $a --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2/bench1.jsonl 2>> gpurun_out/r2/bench1.err
done
