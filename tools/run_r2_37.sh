mkdir -p gpurun_out/r2
FGF_FUZZ_SEEDS=3000 FGF_FUZZ_BAND_SEEDS=600 timeout 2400 python -m pytest tests/test_fuzz_gpu.py -q -p no:cacheprovider > gpurun_out/r2/fuzz37.log 2>&1; echo rc=$? >> gpurun_out/r2/fuzz37.log
timeout 900 python -m pytest tests/test_bands_gpu.py tests/test_report_gpu.py -q -p no:cacheprovider >> gpurun_out/r2/fuzz37.log 2>&1; echo rc=$? >> gpurun_out/r2/fuzz37.log
