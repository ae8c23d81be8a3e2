mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench29.jsonl; rm -f $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for v in 1 2 3 1; do echo "v $v" >> gpurun_out/r2/bench29.err
  FGF_DEV=1 FGF_WIDE_V=$v timeout 300 python bench.py --config 4 --s 1 --batch 32 $B >> $O 2>> gpurun_out/r2/bench29.err
  FGF_DEV=1 FGF_WIDE_V=$v timeout 300 python bench.py --config 1 --s 1 $B >> $O 2>> gpurun_out/r2/bench29.err
done
