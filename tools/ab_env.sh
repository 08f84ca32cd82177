#!/bin/bash
# usage: tools/ab_env.sh tag "ENV=val ..." "configs"   -- bench A (no env) vs B (env) back to back
tag=$1; envs=$2; cfgs=${3:-C2}; out=gpurun_out/$tag; mkdir -p $out
for c in $cfgs; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --others "" > $out/bench_A_$c.json 2> $out/A_$c.err
  env $envs timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --others "" > $out/bench_B_$c.json 2> $out/B_$c.err
done
