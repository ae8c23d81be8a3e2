mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "tiny or graph" > gpurun_out/r2/t18.log 2>&1; echo rc=$? >> gpurun_out/r2/t18.log
O=gpurun_out/r2/bench18.jsonl; rm -f $O
B="--steps 50 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py --config 0 $B >> $O 2>> gpurun_out/r2/bench18.err
A="--config 0 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
python bench.py $A > gpurun_out/r2/p18.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tiny -s 2 -c 1 -o gpurun_out/r2/k6b_cfg0 python bench.py $A > gpurun_out/r2/ncu18.log 2>&1
