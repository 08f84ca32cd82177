#!/bin/bash
# usage: tools/gpu_launch.sh tag "configs"  -- ncu launch lists (duration + DRAM bytes), 4 iterations
tag=${1:-l}; out=gpurun_out/$tag; mkdir -p $out
for cfg in $2; do
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $out/launches_$cfg.csv python tools/run_solve.py --config $cfg --precision fp32,fp64 --reps 1 --niter 4 > $out/launch_$cfg.log 2>&1
done
