mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "graph" > gpurun_out/r2/graph8.log 2>&1; echo rc=$? >> gpurun_out/r2/graph8.log
rm -f gpurun_out/r2/report8.jsonl
FGF_REPORT=gpurun_out/r2/report8.jsonl timeout 900 python -m pytest tests/test_report_gpu.py -x -q > gpurun_out/r2/report8.log 2>&1; echo rc=$? >> gpurun_out/r2/report8.log
