# A/B/C of library builds on one box (bench lines, K13 time): bash tools/run_ab3.sh <tag> "<libs>" "<bench args>;..."
set -u
T=$1; LIBS=$2; IFS=';' read -ra CFGS <<< "$3"
O=gpurun_out/$T; mkdir -p $O
for r in 1 2; do
  for i in "${!CFGS[@]}"; do
    for L in $LIBS; do
      FGF_LIB_NAME=$L python bench.py ${CFGS[$i]} --no-e2e --no-cpu-baseline > $O/c${i}_${L%.so}_$r.json 2>>$O/err.log
      python -c "import json,sys; d=json.load(open('$O/c${i}_${L%.so}_$r.json')); k=d['kernels']; print('$L', '${CFGS[$i]}', round(d['ms_per_step'],4), {n: round(v['ms_per_launch'],4) for n, v in k.items() if v['ms_per_launch']})"
    done
  done
done
