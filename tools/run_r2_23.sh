E=gpurun_out/ev4; mkdir -p $E
python tools/config_calls.py > $E/calls.json 2> $E/calls.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k 'regex:output|lowres|box_strip|subsample|wide|tiny' --csv --log-file $E/launches_configs.csv \
  python tools/config_calls.py > $E/ncu_configs.log 2>&1 && \
python tools/ncu_bytes.py $E/launches_configs.csv $E/calls.json $E/ncu_bytes.json > $E/ncu_bytes.log 2>&1
FGF_NCU_BYTES=$E/ncu_bytes.json FGF_REPORT=$E/report.jsonl timeout 900 python -m pytest tests/test_report_gpu.py -q > $E/report.log 2>&1
