#!/bin/bash
# usage: tools/ab_lib.sh tag "build_ab/libX.so ..." "C5 C3"  -- short bench of the default library and
# of each variant build (NBK_LIB), interleaved twice, same box
tag=$1; libs=$2; cfgs=${3:-C5}; out=gpurun_out/$tag; mkdir -p $out
for rep in 1 2; do
for c in $cfgs; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study \
    --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/A_${c}_$rep.json 2> $out/A_${c}_$rep.err
  for l in $libs; do
    b=$(basename $l .so)
    NBK_LIB=$l timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study \
      --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/${b}_${c}_$rep.json 2> $out/${b}_${c}_$rep.err
  done
done
done
