set -u
O=gpurun_out/pdl2; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_apps_gpu.py tests/test_halfio_gpu.py tests/test_u8io_gpu.py tests/test_fuzz_gpu.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for r in 1 2; do
  for L in libfgf_base.so libfgf.so; do
    FGF_LIB_NAME=$L python bench.py --config 2 --steps 200 --no-e2e --no-cpu-baseline > $O/c2_${L%.so}_$r.json 2>>$O/err.log
    FGF_LIB_NAME=$L python bench.py --config 3 --steps 30 --no-e2e --no-cpu-baseline > $O/c3_${L%.so}_$r.json 2>>$O/err.log
  done
done
