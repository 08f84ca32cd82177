#!/bin/bash
# parity subset (incl. full-size C3 / C5 CG) + one C5 bench line of the in-tree build
out=gpurun_out/${1:-verify}; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pcg.py tests/test_gpu_single.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py tests/test_gpu_api.py -x -q > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/bench_C5.json 2> $out/bench_C5.err
