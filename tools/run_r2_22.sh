mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_apps_gpu.py tests/test_abi.py -q > gpurun_out/r2/t22.log 2>&1; echo rc=$? >> gpurun_out/r2/t22.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke22.log 2>&1; echo rc=$? >> gpurun_out/r2/smoke22.log
