mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench25.jsonl; rm -f $O
B="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
for tw in 128 160 192 224 256; do echo "c4 tw $tw" >> gpurun_out/r2/bench25.err
  FGF_DEV=1 FGF_WIDE_TW=$tw timeout 300 python bench.py --config 4 --s 1 --batch 32 $B >> $O 2>> gpurun_out/r2/bench25.err; done
for tw in 160 224 256 288 320; do echo "c1 tw $tw" >> gpurun_out/r2/bench25.err
  FGF_DEV=1 FGF_WIDE_TW=$tw timeout 300 python bench.py --config 1 --s 1 $B >> $O 2>> gpurun_out/r2/bench25.err; done
for v in 0 1; do for tw in 160 256 320; do echo "c4s2 v $v tw $tw" >> gpurun_out/r2/bench25.err
  FGF_DEV=1 FGF_WIDE_V=$v FGF_WIDE_TW=$tw timeout 300 python bench.py --config 4 --s 2 --batch 64 $B >> $O 2>> gpurun_out/r2/bench25.err; done; done
