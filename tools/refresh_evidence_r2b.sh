#!/bin/bash
# Round-2 final evidence on one GPU (run under gpurun): bench lines, ncu launch lists, full
# captures of every engine's kernel with stall reasons, per-config report with B_ncu.
# Output: gpurun_out/ev3/ (copied to profiles/round2/ by hand).
set -u
E=gpurun_out/${EV:-ev3}; mkdir -p $E
NB="--no-e2e --no-cpu-baseline"
timeout 900 python -m pytest tests -m gpu -x -q > $E/pytest_gpu.log 2>&1; echo rc=$? >> $E/pytest_gpu.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $E/smi.txt 2>&1
python bench.py > $E/bench.json 2> $E/bench.err || { tail -5 $E/bench.err; exit 1; }
for a in "--config 4 --s 1 --batch 32" "--config 4 --s 2" "--config 4 --s 8" "--config 1 --s 1" \
         "--config 0" "--config 1" "--config 2" "--config 3" "--config 5" "--dtype f16" "--dtype u8"; do
  timeout 600 python bench.py $a --steps 20 --warmup 3 $NB >> $E/bench_lines.jsonl 2>> $E/bench_lines.err
done
# launch list of the default bench command (K4 / K13 shares and DRAM bytes per launch)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k 'regex:output|lowres|box_strip|subsample|wide|tiny' --csv --log-file $E/launches_cfg4.csv \
  python bench.py --steps 2 --warmup 3 $NB > $E/ncu_launches.log 2>&1
python tools/launch_summary.py $E/launches_cfg4.csv > $E/launches_cfg4_summary.txt 2>&1
# per-config launch list (one warm-up + one measured call per report record) -> B_ncu
python tools/config_calls.py > $E/calls.json 2> $E/calls.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k 'regex:output|lowres|box_strip|subsample|wide|tiny' --csv --log-file $E/launches_configs.csv \
  python tools/config_calls.py > $E/ncu_configs.log 2>&1 && \
python tools/ncu_bytes.py $E/launches_configs.csv $E/calls.json $E/ncu_bytes.json > $E/ncu_bytes.log 2>&1
FGF_NCU_BYTES=$E/ncu_bytes.json FGF_REPORT=$E/report.jsonl timeout 900 python -m pytest tests/test_report_gpu.py -q > $E/report.log 2>&1
full() {  # name, kernel regex, extra ncu args, bench args
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" $3 \
    -o $E/$1 python bench.py $4 $NB > $E/ncu_$1.log 2>&1
  python tools/ncu_summary.py $E/$1.ncu-rep > $E/$1_summary.txt 2>&1
  for k in 0 1 2 3 4 5; do python tools/ncu_phases.py $E/$1.ncu-rep $k >> $E/$1_phases.txt 2>&1 || break; done
  rm -f $E/$1.ncu-rep
}
full full_cfg4 'lowres|output' '-s 2 -c 2' '--batch 16 --steps 2 --warmup 1'
full full_k5_cfg1_s1 wide '-s 2 -c 1' '--config 1 --s 1 --steps 2 --warmup 1'
full full_k5_cfg4_s2 wide '-s 2 -c 1' '--config 4 --s 2 --batch 8 --steps 2 --warmup 1'
full full_cfg3 'subsample|box_strip|output' '-s 5 -c 5' '--config 3 --batch 8 --steps 2 --warmup 1'
full full_k6_cfg0 tiny '-s 2 -c 1' '--config 0 --steps 2 --warmup 1'
full full_cfg1 'lowres|output' '-s 4 -c 2' '--config 1 --steps 2 --warmup 1'
du -sh $E
echo done
