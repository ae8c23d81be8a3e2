#!/bin/bash
# Round-2 closing evidence on one GPU (run under gpurun), HEAD's build: the GPU suite, the
# default bench line, every other workload's bench line, the driver's torchrun launch with one
# rank (NCCL process group, max-over-ranks reduction), the reference arm, and the ncu launch
# list of the default bench command.  The ncu full captures of profiles/round2/ are of the same
# kernels (no kernel source changed since) and are not repeated.  Output: gpurun_out/ev7/.
set -u
E=gpurun_out/${EV:-ev7}; mkdir -p $E
NB="--no-e2e --no-cpu-baseline"
timeout 900 python -m pytest tests -m gpu -x -q > $E/pytest_gpu.log 2>&1; echo rc=$? >> $E/pytest_gpu.log
tail -3 $E/pytest_gpu.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $E/smi.txt 2>&1
python bench.py > $E/bench.json 2> $E/bench.err || { tail -5 $E/bench.err; exit 1; }
cut -c1-300 $E/bench.json
for a in "--config 4 --s 1 --batch 32" "--config 4 --s 2" "--config 4 --s 8" "--config 1 --s 1" \
         "--config 0" "--config 1" "--config 2" "--config 3" "--config 5" "--dtype f16" "--dtype u8" \
         "--config 0 --graph" "--config 1 --graph"; do
  timeout 600 python bench.py $a --steps 20 --warmup 3 $NB >> $E/bench_lines.jsonl 2>> $E/bench_lines.err
done
# the driver's multi-GPU launch line, one rank (all this pool has): NCCL init, barrier, MAX reduce
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 1 --steps 10 --warmup 3 $NB > $E/bench_torchrun1.json 2> $E/bench_torchrun1.err
echo torchrun rc=$?; cut -c1-200 $E/bench_torchrun1.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $E/bench_reference.json 2> $E/bench_reference.err
echo reference rc=$?; cut -c1-300 $E/bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k 'regex:output|lowres|box_strip|subsample|wide|tiny' --csv --log-file $E/launches_cfg4.csv \
  python bench.py --steps 2 --warmup 3 $NB > $E/ncu_launches.log 2>&1
python tools/launch_summary.py $E/launches_cfg4.csv > $E/launches_cfg4_summary.txt 2>&1
tail -8 $E/launches_cfg4_summary.txt
du -sh $E
echo done
