# A/B of the L2 prefetch of the guidance under K13 (single images): FGF_NO_L2PF=1 turns it off
O=gpurun_out/l2pf; mkdir -p $O
for r in 1 2 3; do
  for knob in 0 1; do
    for cfg in "--config 1 --steps 200" "--config 1 --steps 200 --graph"; do
      if [ $knob = 1 ]; then E="FGF_DEV=1 FGF_NO_L2PF=1"; else E="FGF_DEV=1"; fi
      env $E python bench.py $cfg --no-e2e --no-cpu-baseline > $O/tmp.json 2>>$O/err.log
      python -c "import json; d=json.load(open('$O/tmp.json')); k=d['kernels']; print('nopf=$knob', '$cfg', round(d['ms_per_step']*1e3,2), 'us', {n: round(v['ms_per_launch']*1e3,2) for n, v in k.items() if v['ms_per_launch']})" | tee -a $O/summary.txt
    done
  done
done
