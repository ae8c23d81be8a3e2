# A/B of two builds of the library on one box: FGF_LIB_NAME selects the .so (bench.py and the
# binding load it); usage: bash tools/run_ab_lib.sh <tag> <lib_a> <lib_b> "<bench args>;<bench args>;..."
set -u
T=$1; A=$2; B=$3; IFS=';' read -ra CFGS <<< "$4"
O=gpurun_out/$T; mkdir -p $O
for r in 1 2; do
  for i in "${!CFGS[@]}"; do
    for L in $A $B; do
      FGF_LIB_NAME=$L python bench.py ${CFGS[$i]} --no-e2e --no-cpu-baseline > $O/c${i}_${L%.so}_$r.json 2>>$O/err.log
    done
  done
done
