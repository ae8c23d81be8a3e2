set -u
O=gpurun_out/nt; mkdir -p $O
for r in 1 2; do
  for nt in 0 96 128 160 192 224; do
    if [ $nt = 0 ]; then FGF_DEV=1 python bench.py --config 1 --steps 200 --no-e2e --no-cpu-baseline > $O/c1_nt${nt}_$r.json 2>>$O/err.log
    else FGF_DEV=1 FGF_LR_NT=$nt python bench.py --config 1 --steps 200 --no-e2e --no-cpu-baseline > $O/c1_nt${nt}_$r.json 2>>$O/err.log; fi
  done
  for nt in 0 128 192; do
    if [ $nt = 0 ]; then FGF_DEV=1 python bench.py --config 5 --steps 20 --no-e2e --no-cpu-baseline > $O/c5_nt${nt}_$r.json 2>>$O/err.log
    else FGF_DEV=1 FGF_LR_NT=$nt python bench.py --config 5 --steps 20 --no-e2e --no-cpu-baseline > $O/c5_nt${nt}_$r.json 2>>$O/err.log; fi
  done
done
