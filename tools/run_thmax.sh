set -u
O=gpurun_out/thmax; mkdir -p $O
for r in 1 2; do
  for t in 0 46 54 64 68 90 135; do
    if [ $t = 0 ]; then python bench.py --config 3 --steps 30 --no-e2e --no-cpu-baseline > $O/c3_t${t}_$r.json 2>>$O/err.log
    else FGF_DEV=1 FGF_STRIP_THMAX=$t python bench.py --config 3 --steps 30 --no-e2e --no-cpu-baseline > $O/c3_t${t}_$r.json 2>>$O/err.log; fi
  done
  for t in 0 25 30 38 50 75; do
    if [ $t = 0 ]; then python bench.py --config 2 --steps 100 --no-e2e --no-cpu-baseline > $O/c2_t${t}_$r.json 2>>$O/err.log
    else FGF_DEV=1 FGF_STRIP_THMAX=$t python bench.py --config 2 --steps 100 --no-e2e --no-cpu-baseline > $O/c2_t${t}_$r.json 2>>$O/err.log; fi
  done
done
