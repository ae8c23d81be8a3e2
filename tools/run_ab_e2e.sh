# e2e A/B of two library builds (FGF_LIB_NAME) on one box
set -u
T=$1; A=$2; B=$3
O=gpurun_out/$T; mkdir -p $O
for r in 1 2; do
  for L in $A $B; do
    FGF_LIB_NAME=$L python bench.py --steps 5 --no-cpu-baseline --e2e-steps 3 > $O/${L%.so}_$r.json 2>>$O/err.log
  done
done
