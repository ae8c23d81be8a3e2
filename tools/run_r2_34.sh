mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench34.jsonl; rm -f $O
B="--steps 30 --warmup 3 --no-e2e --no-cpu-baseline"
for k in 0 1 0 1; do echo "inplace $k" >> gpurun_out/r2/bench34.err
  if [ $k = 1 ]; then FGF_DEV=1 FGF_STRIP_INPLACE=1 timeout 300 python bench.py --config 2 $B >> $O 2>> gpurun_out/r2/bench34.err;
  else timeout 300 python bench.py --config 2 $B >> $O 2>> gpurun_out/r2/bench34.err; fi
done
FGF_DEV=1 FGF_STRIP_INPLACE=1 timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "config_single" > gpurun_out/r2/t34.log 2>&1; echo rc=$? >> gpurun_out/r2/t34.log
