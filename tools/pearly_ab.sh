out=gpurun_out/pe; mkdir -p $out
for rep in 1 2; do for v in 1 0; do for c in C2 C5 C3; do
NBK_P_EARLY=$v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --others "" --no-jacobi --no-accuracy --no-precision-study > $out/b_${v}_${c}_$rep.json 2>$out/b_${v}_${c}_$rep.err
done; done; done
