mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/gputest7.log 2>&1; echo rc=$? >> gpurun_out/r2/gputest7.log
O=gpurun_out/r2/bench7.jsonl; rm -f $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for a in "--config 4 --s 1 --batch 32" "--config 1 --s 1" "--config 4 --s 2 --batch 64" "--config 4 --s 8 --batch 64"; do
  timeout 300 python bench.py $a $B >> $O 2>> gpurun_out/r2/bench7.err
done
timeout 300 python bench.py --steps 20 --warmup 3 >> $O 2>> gpurun_out/r2/bench7.err
