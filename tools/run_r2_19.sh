mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench19.jsonl; rm -f $O
B="--steps 50 --warmup 3 --no-e2e --no-cpu-baseline"
for r in 4 8 16 32; do echo "rows $r" >> gpurun_out/r2/bench19.err
  FGF_DEV=1 FGF_TINY_ROWS=$r timeout 300 python bench.py --config 0 $B >> $O 2>> gpurun_out/r2/bench19.err
done
timeout 300 python bench.py --config 0 $B >> $O 2>> gpurun_out/r2/bench19.err
