mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench6.jsonl; rm -f $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for v in 0 1; do
for a in "--config 4 --s 1 --batch 32" "--config 1 --s 1" "--config 4 --s 2 --batch 64"; do
  FGF_DEV=1 FGF_WIDE_V=$v timeout 300 python bench.py $a $B >> $O 2>> gpurun_out/r2/bench6.err
done; done
FGF_DEV=1 FGF_WIDE_TW=320 timeout 300 python bench.py --config 1 --s 1 $B >> $O 2>> gpurun_out/r2/bench6.err
FGF_DEV=1 FGF_WIDE_TW=320 FGF_WIDE_V=1 timeout 300 python bench.py --config 1 --s 1 $B >> $O 2>> gpurun_out/r2/bench6.err
FGF_DEV=1 FGF_ENGINE=strip timeout 300 python bench.py --config 1 --s 1 $B >> $O 2>> gpurun_out/r2/bench6.err
FGF_DEV=1 FGF_ENGINE=strip timeout 300 python bench.py --config 4 --s 1 --batch 32 $B >> $O 2>> gpurun_out/r2/bench6.err
