mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_bands_gpu.py -x -q > gpurun_out/r2/bands10.log 2>&1; echo rc=$? >> gpurun_out/r2/bands10.log
O=gpurun_out/r2/bench10.jsonl; rm -f $O
timeout 300 python bench.py --config 5 --steps 20 --warmup 3 >> $O 2>> gpurun_out/r2/bench10.err
timeout 300 python bench.py --config 5 --band-mode two-step --steps 20 --warmup 3 >> $O 2>> gpurun_out/r2/bench10.err
