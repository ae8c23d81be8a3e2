# K5 variant sweep (FGF_WIDE_V) on one box: bash tools/run_wide_v.sh <tag> "<bench args>;..."
set -u
T=$1; IFS=';' read -ra CFGS <<< "$2"
O=gpurun_out/$T; mkdir -p $O
for r in 1 2; do
  for i in "${!CFGS[@]}"; do
    for v in 0 1 2 3; do
      FGF_DEV=1 FGF_WIDE_V=$v python bench.py ${CFGS[$i]} --no-e2e --no-cpu-baseline > $O/c${i}_v${v}_$r.json 2>>$O/err.log
    done
  done
done
