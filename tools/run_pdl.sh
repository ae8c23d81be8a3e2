set -u
O=gpurun_out/pdl1; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for r in 1 2; do
  for L in libfgf_base.so libfgf.so; do
    FGF_LIB_NAME=$L python bench.py --config 1 --steps 300 --no-e2e --no-cpu-baseline > $O/c1_${L%.so}_$r.json 2>>$O/err.log
    FGF_LIB_NAME=$L python bench.py --config 5 --steps 30 --no-e2e --no-cpu-baseline > $O/c5_${L%.so}_$r.json 2>>$O/err.log
    FGF_LIB_NAME=$L python bench.py --config 4 --s 8 --batch 8 --steps 50 --no-e2e --no-cpu-baseline > $O/c48_${L%.so}_$r.json 2>>$O/err.log
  done
  FGF_DEV=1 FGF_NO_PDL=1 python bench.py --config 1 --steps 300 --no-e2e --no-cpu-baseline > $O/c1_nopdl_dev_$r.json 2>>$O/err.log
  FGF_DEV=1 python bench.py --config 1 --steps 300 --no-e2e --no-cpu-baseline > $O/c1_pdl_dev_$r.json 2>>$O/err.log
done
python bench.py --no-e2e --no-cpu-baseline > $O/c4_new.json 2>>$O/err.log
