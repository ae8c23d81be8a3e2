mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench20.jsonl; rm -f $O
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py --config 4 --s 2 --batch 64 $B >> $O 2>> gpurun_out/r2/bench20.err
FGF_DEV=1 FGF_WIDE_COMPACT=1 timeout 300 python bench.py --config 4 --s 2 --batch 64 $B >> $O 2>> gpurun_out/r2/bench20.err
FGF_DEV=1 FGF_WIDE_COMPACT=1 FGF_WIDE_BULK=1 timeout 300 python bench.py --config 4 --s 2 --batch 64 $B >> $O 2>> gpurun_out/r2/bench20.err
FGF_DEV=1 FGF_WIDE_COMPACT=1 FGF_WIDE_V=1 timeout 300 python bench.py --config 4 --s 2 --batch 64 $B >> $O 2>> gpurun_out/r2/bench20.err
timeout 300 python bench.py --config 0 --steps 50 --warmup 3 --no-e2e --no-cpu-baseline >> $O 2>> gpurun_out/r2/bench20.err
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k tiny > gpurun_out/r2/t20.log 2>&1
