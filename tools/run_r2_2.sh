mkdir -p gpurun_out/r2
A="--config 1 --s 1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
python bench.py $A > gpurun_out/r2/p4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wide -s 2 -c 1 -o gpurun_out/r2/k5v2_cfg1 python bench.py $A > gpurun_out/r2/ncu4.log 2>&1
echo rc=$? >> gpurun_out/r2/ncu4.log
