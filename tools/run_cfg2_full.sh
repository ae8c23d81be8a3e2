set -u
E=gpurun_out/ev5; mkdir -p $E
NB="--no-e2e --no-cpu-baseline"
full() {  # name, kernel regex, extra ncu args, bench args
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" $3 \
    -o $E/$1 python bench.py $4 $NB > $E/ncu_$1.log 2>&1
  python tools/ncu_summary.py $E/$1.ncu-rep > $E/$1_summary.txt 2>&1
  for k in 0 1 2 3 4 5; do python tools/ncu_phases.py $E/$1.ncu-rep $k >> $E/$1_phases.txt 2>&1 || break; done
  rm -f $E/$1.ncu-rep
}
# config 2: one 4000 x 3000 colour frame, r' = 15 (the strip engine at a wide window)
full full_cfg2 'subsample|box_strip|output' '-s 5 -c 5' '--config 2 --steps 2 --warmup 1'
# config 4 at s = 2 through the strip engine (r' = 16; FGF_ENGINE=strip) for comparison with K5
FGF_DEV=1 FGF_ENGINE=strip timeout 600 ncu --set full --clock-control none -k "regex:box_strip" -s 2 -c 2 \
  -o $E/full_strip_cfg4_s2 python bench.py --config 4 --s 2 --batch 8 --steps 2 --warmup 1 $NB > $E/ncu_strip.log 2>&1
python tools/ncu_summary.py $E/full_strip_cfg4_s2.ncu-rep > $E/full_strip_cfg4_s2_summary.txt 2>&1; rm -f $E/full_strip_cfg4_s2.ncu-rep
FGF_DEV=1 FGF_ENGINE=strip python bench.py --config 4 --s 2 --steps 5 $NB > $E/strip_cfg4_s2.json 2>&1
