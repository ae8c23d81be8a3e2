mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_wide_gpu.py -x -q > gpurun_out/r2/t26.log 2>&1; echo rc=$? >> gpurun_out/r2/t26.log
O=gpurun_out/r2/bench26.jsonl; rm -f $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for kc in 0 1 2; do echo "kc $kc" >> gpurun_out/r2/bench26.err
  for a in "--config 4 --s 1 --batch 32" "--config 1 --s 1"; do
    if [ $kc = 0 ]; then timeout 300 python bench.py $a $B >> $O 2>> gpurun_out/r2/bench26.err;
    else FGF_DEV=1 FGF_WIDE_KC=$kc timeout 300 python bench.py $a $B >> $O 2>> gpurun_out/r2/bench26.err; fi
  done
done
