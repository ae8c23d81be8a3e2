set -u
O=gpurun_out/exp6; mkdir -p $O
timeout 300 python -m pytest tests/test_lowres_fused_gpu.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for r in 1 2; do
  python bench.py --no-e2e --no-cpu-baseline > $O/def_$r.json 2>>$O/err.log
  FGF_DEV=1 FGF_LR_V=4 python bench.py --no-e2e --no-cpu-baseline > $O/v4_$r.json 2>>$O/err.log
  python bench.py --config 1 --steps 200 --no-e2e --no-cpu-baseline > $O/c1def_$r.json 2>>$O/err.log
  FGF_DEV=1 FGF_LR_V=4 python bench.py --config 1 --steps 200 --no-e2e --no-cpu-baseline > $O/c1v4_$r.json 2>>$O/err.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:output" -s 1 -c 1 \
  -o $O/k4c python bench.py --config 3 --batch 8 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_k4c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:lowres" -s 1 -c 1 \
  -o $O/k13v4 env FGF_DEV=1 FGF_LR_V=4 python bench.py --batch 16 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_k13v4.log 2>&1
