mkdir -p gpurun_out/r2
O=gpurun_out/r2/bench33.jsonl; rm -f $O
B="--steps 30 --warmup 3 --no-e2e --no-cpu-baseline"
for hp in 24 16 12 8 24; do echo "hpre $hp" >> gpurun_out/r2/bench33.err
  FGF_DEV=1 FGF_HPRE_R=$hp timeout 300 python bench.py --config 2 $B >> $O 2>> gpurun_out/r2/bench33.err
done
for th in 64 32 128 16; do echo "thmax $th" >> gpurun_out/r2/bench33.err
  FGF_DEV=1 FGF_STRIP_THMAX=$th timeout 300 python bench.py --config 2 $B >> $O 2>> gpurun_out/r2/bench33.err
done
