out=gpurun_out/pdl; mkdir -p $out
for m in 0 1 4 5 7; do
  for c in C2 C4; do
    NBK_PDL=$m timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --others "" --no-jacobi --no-accuracy --no-precision-study > $out/b_${m}_$c.json 2>/dev/null
  done
done
