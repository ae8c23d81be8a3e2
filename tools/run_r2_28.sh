mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2/gputest28.log 2>&1; echo rc=$? >> gpurun_out/r2/gputest28.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke28.log 2>&1; echo rc=$? >> gpurun_out/r2/smoke28.log
python bench.py > gpurun_out/r2/bench28.json 2> gpurun_out/r2/bench28.err
for a in "--config 4 --s 2 --batch 64" "--config 4 --s 2 --batch 64" "--config 4 --s 1 --batch 32"; do
  timeout 300 python bench.py $a --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2/bench28b.jsonl 2>> gpurun_out/r2/bench28.err
done
