#!/bin/bash
# Round-end evidence on one GPU (run under gpurun): bench line, ncu launch list of the same
# command, one full capture of K13 and K4 at the bench configuration, per-config report.
set -u
mkdir -p gpurun_out/ev
python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err || { tail -5 gpurun_out/ev/bench.err; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k 'regex:output|lowres|box_strip|subsample' --csv --log-file gpurun_out/ev/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:lowres_gray|output_async' -c 2 \
  -o gpurun_out/ev/full_cfg4 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > gpurun_out/ev/ncu_full.log 2>&1
FGF_REPORT=gpurun_out/ev/report.jsonl timeout 900 python -m pytest tests/test_report_gpu.py -q 2>&1 | tail -1
