mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench9.jsonl; rm -f $O
B="--steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
for mb in 8192 200 100 48 24; do
  echo "chunk $mb" >> gpurun_out/r2/bench9.err
  FGF_DEV=1 FGF_CHUNK_MB=$mb timeout 300 python bench.py --config 3 $B >> $O 2>> gpurun_out/r2/bench9.err
done
for e in k13 wide; do
  FGF_DEV=1 FGF_ENGINE=$e timeout 300 python bench.py --config 1 $B >> $O 2>> gpurun_out/r2/bench9.err
  FGF_DEV=1 FGF_ENGINE=$e timeout 300 python bench.py --config 0 $B >> $O 2>> gpurun_out/r2/bench9.err
done
timeout 300 python bench.py --config 2 $B >> $O 2>> gpurun_out/r2/bench9.err
