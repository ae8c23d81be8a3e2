mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench14.jsonl; rm -f $O
B="--steps 30 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 python -m pytest tests/test_wide_gpu.py -x -q > gpurun_out/r2/wide14.log 2>&1; echo rc=$? >> gpurun_out/r2/wide14.log
for a in "--config 4 --s 1 --batch 32" "--config 1 --s 1" "--config 4 --s 2 --batch 64"; do
  timeout 300 python bench.py $a $B >> $O 2>> gpurun_out/r2/bench14.err
done
for th in 8 16 32 64; do for nt in 96 160; do
  echo "TH $th NT $nt" >> gpurun_out/r2/bench14.err
  FGF_DEV=1 FGF_LR_TH=$th FGF_LR_NT=$nt timeout 300 python bench.py --config 1 $B >> $O 2>> gpurun_out/r2/bench14.err
done; done
for tr in 4 8 16 32; do
  echo "TR $tr" >> gpurun_out/r2/bench14.err
  FGF_DEV=1 FGF_K4_TR=$tr timeout 300 python bench.py --config 1 $B >> $O 2>> gpurun_out/r2/bench14.err
done
