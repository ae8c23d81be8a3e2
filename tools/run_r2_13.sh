mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_lowres_fused_gpu.py -x -q > gpurun_out/r2/k13_13.log 2>&1; echo rc=$? >> gpurun_out/r2/k13_13.log
A="--config 1 --s 1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
python bench.py $A > gpurun_out/r2/p13.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wide -s 2 -c 1 -o gpurun_out/r2/k5v1_cfg1 python bench.py $A > gpurun_out/r2/ncu13.log 2>&1
echo rc=$? >> gpurun_out/r2/ncu13.log
O=gpurun_out/r2/bench13.jsonl; rm -f $O
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline >> $O 2>> gpurun_out/r2/bench13.err; done
