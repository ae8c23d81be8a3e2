mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_wide_gpu.py -x -q > gpurun_out/r2/t27.log 2>&1; echo rc=$? >> gpurun_out/r2/t27.log
O=gpurun_out/r2/bench27.jsonl; rm -f $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py --config 4 --s 1 --batch 32 $B >> $O 2>> gpurun_out/r2/bench27.err
FGF_DEV=1 FGF_WIDE_TW=256 timeout 300 python bench.py --config 4 --s 1 --batch 32 $B >> $O 2>> gpurun_out/r2/bench27.err
timeout 300 python bench.py --config 1 --s 1 $B >> $O 2>> gpurun_out/r2/bench27.err
timeout 300 python bench.py --config 4 --s 2 --batch 64 $B >> $O 2>> gpurun_out/r2/bench27.err
