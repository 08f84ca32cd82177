# Warm-cache DRAM traffic of the steady-state kernels (ncu --cache-control none):
# does the C2 working set stay in L2 across CG iterations?
out=gpurun_out/warm; mkdir -p $out
for cfg in C2 C4; do
timeout 600 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv \
  --log-file $out/warm_$cfg.csv python tools/run_solve.py --config $cfg --precision fp32,fp64 --reps 1 --niter 12 > $out/warm_$cfg.log 2>&1
done
