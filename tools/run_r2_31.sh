mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench31.jsonl; rm -f $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for lib in libfgf.so libfgf_prekc.so libfgf.so libfgf_prekc.so; do echo "lib $lib" >> gpurun_out/r2/bench31.err
  FGF_LIB_NAME=$lib timeout 300 python bench.py --config 4 --s 2 --batch 64 $B >> $O 2>> gpurun_out/r2/bench31.err
done
