#!/bin/bash
out=gpurun_out/r2l; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
for rep in 1 2; do
for c in C5 C3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/A_${c}_$rep.json 2> $out/A_${c}_$rep.err
  NBK_LIB=build_ab/libnbk_epb1.so timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/EPB1_${c}_$rep.json 2> $out/EPB1_${c}_$rep.err
  for pdl in 3 5 7; do
    NBK_PDL=$pdl timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/PDL${pdl}_${c}_$rep.json 2> $out/PDL${pdl}_${c}_$rep.err
  done
done
done
