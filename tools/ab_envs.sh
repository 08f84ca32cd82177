#!/bin/bash
# usage: tools/ab_envs.sh tag "C5 C4" "ENV1=a ENV2=b" "ENV1=c" ...  -- short bench per env setting
# (the first run has no extra env), interleaved twice on the same box
tag=$1; cfgs=$2; shift 2; out=gpurun_out/$tag; mkdir -p $out
for rep in 1 2; do
for c in $cfgs; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study \
    --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/A_${c}_$rep.json 2> $out/A_${c}_$rep.err
  i=0
  for envs in "$@"; do
    i=$((i+1))
    env $envs timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study \
      --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/E${i}_${c}_$rep.json 2> $out/E${i}_${c}_$rep.err
    echo "E$i: $envs" > $out/E${i}.env
  done
done
done
