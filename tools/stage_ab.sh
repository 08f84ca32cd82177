# K_B index staging A/B (NBK_DSSUM_STAGE runtime switch) + GPU tests
out=gpurun_out/stg2; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
for st in 1 0; do for c in C2 C4 C3; do
NBK_DSSUM_STAGE=$st timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --others "" --no-jacobi --no-accuracy --no-precision-study > $out/b_${st}_$c.json 2>$out/b_${st}_$c.err
done; done
