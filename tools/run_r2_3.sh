mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_wide_gpu.py -x -q > gpurun_out/r2/wide5.log 2>&1; echo rc=$? >> gpurun_out/r2/wide5.log
rm -f gpurun_out/r2/bench5.jsonl
for a in "--config 4 --s 1 --batch 32" "--config 1 --s 1" "--config 4 --s 2 --batch 64"; do
  timeout 300 python bench.py $a --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2/bench5.jsonl 2>> gpurun_out/r2/bench5.err
done
FGF_DEV=1 FGF_ENGINE=wide timeout 300 python bench.py --config 4 --s 4 --batch 64 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2/bench5.jsonl 2>> gpurun_out/r2/bench5.err
timeout 300 python bench.py --config 4 --s 4 --batch 64 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2/bench5.jsonl 2>> gpurun_out/r2/bench5.err
