#!/bin/bash
out=gpurun_out/r2k; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for rep in 1 2; do
for c in C5 C4 C2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/A_${c}_$rep.json 2> $out/A_${c}_$rep.err
  NBK_LIB=build_ab/libnbk_kb4.so timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/KB4_${c}_$rep.json 2> $out/KB4_${c}_$rep.err
  NBK_LIB=build_ab/libnbk_kb4.so NBK_DSSUM_TILE_NODES=1024 timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/KB4t1024_${c}_$rep.json 2> $out/KB4t1024_${c}_$rep.err
done
done
