set -u
O=gpurun_out/ab2; mkdir -p $O
for i in 1 2; do
  python bench.py --no-e2e --no-cpu-baseline > $O/bulk_$i.json 2>>$O/err.log
  FGF_DEV=1 FGF_LR_NOBULK=1 python bench.py --no-e2e --no-cpu-baseline > $O/nobulk_$i.json 2>>$O/err.log
done
for c in 1; do
  python bench.py --config $c --no-e2e --no-cpu-baseline --steps 200 > $O/cfg${c}_bulk.json 2>>$O/err.log
  FGF_DEV=1 FGF_LR_NOBULK=1 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 200 > $O/cfg${c}_nobulk.json 2>>$O/err.log
done
timeout 300 python -m pytest tests/test_lowres_fused_gpu.py tests/test_parity_gpu.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
