set -u
O=gpurun_out/k4tr; mkdir -p $O
for r in 1 2; do
  for tr in 0 4 16 32; do
    if [ $tr = 0 ]; then FGF_DEV=1 python bench.py --config 1 --steps 300 --no-e2e --no-cpu-baseline > $O/c1_tr${tr}_$r.json 2>>$O/err.log
    else FGF_DEV=1 FGF_K4_TR=$tr python bench.py --config 1 --steps 300 --no-e2e --no-cpu-baseline > $O/c1_tr${tr}_$r.json 2>>$O/err.log; fi
  done
done
