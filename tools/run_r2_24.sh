E=gpurun_out/k13src; mkdir -p $E
A="--batch 16 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
python bench.py $A > $E/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lowres_gray -c 1 -o $E/k13 python bench.py $A > $E/ncu.log 2>&1
ncu -i $E/k13.ncu-rep --page source --csv --print-source cuda > $E/k13_cuda_src.csv 2>&1
ncu -i $E/k13.ncu-rep --page source --csv > $E/k13_sass.csv 2>&1
python tools/ncu_phases.py $E/k13.ncu-rep 0 > $E/k13_phases.txt 2>&1
gzip -f $E/k13_sass.csv $E/k13_cuda_src.csv
rm -f $E/k13.ncu-rep
ls -la $E
