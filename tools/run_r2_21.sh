mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2/gputest21.log 2>&1; echo rc=$? >> gpurun_out/r2/gputest21.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke21.log 2>&1; echo rc=$? >> gpurun_out/r2/smoke21.log
