#!/bin/bash
out=gpurun_out/${1:-e2e}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_bench.py -x -q > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
timeout 900 python bench.py --config C5 --steps 6 --warmup 3 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/bench_C5.json 2> $out/bench_C5.err
