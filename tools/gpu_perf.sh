#!/bin/bash
# usage: tools/gpu_perf.sh tag "C5 C3" [pytest -k expr]  -- quick parity subset + short bench lines
tag=${1:-perf}; cfgs=${2:-C5}; out=gpurun_out/$tag; mkdir -p $out
if [ -n "$3" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$3" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
fi
for c in $cfgs; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study \
    --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/bench_$c.json 2> $out/bench_$c.err
done
