#!/bin/bash
# usage: tools/gpu_quick.sh tag "configs" [pytest-k]   (runs gpu tests, then bench per config)
tag=${1:-t}; cfgs=${2:-C2}; out=gpurun_out/$tag; mkdir -p $out
if [ -n "$3" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -k "$3" > $out/pytest_gpu.log 2>&1; 
else timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; fi
echo "pytest rc=$?" >> $out/pytest_gpu.log
for c in $cfgs; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --others "" --no-precision-study > $out/bench_$c.json 2> $out/bench_$c.err
done
