#!/bin/bash
# usage: tools/gpu_tests.sh tag [pytest -k expr]
tag=${1:-t}; out=gpurun_out/$tag; mkdir -p $out
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 1200 python -m pytest tests -m gpu -x -q $K > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_C2.json 2> $out/bench_C2.err
