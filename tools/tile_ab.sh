out=gpurun_out/tile; mkdir -p $out
for tn in 0 1024; do
  for c in C2 C4; do
    if [ $tn = 0 ]; then unset NBK_DSSUM_TILE_NODES; else export NBK_DSSUM_TILE_NODES=$tn; fi
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --others "" --no-jacobi --no-accuracy --no-precision-study > $out/b_${tn}_$c.json 2>/dev/null
  done
done
