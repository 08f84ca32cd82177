#!/bin/bash
# FP64 k_axl at N = 12 (8 N^3 shared memory) and N = 8 (one element per CTA): parity + A/B
out=gpurun_out/ab4; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pcg.py tests/test_gpu_single.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -x -q > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
NBK_LIB=build_ab/lib8d.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pcg.py -x -q > $out/pytest_8d.log 2>&1; echo rc=$? >> $out/pytest_8d.log
tail -3 $out/pytest.log
tools/ab_envs.sh ab4/ab "C3 C4 C5" "NBK_LIB=build_ab/libno12.so" "NBK_LIB=build_ab/lib8d.so" "NBK_LIB=build_ab/lib7.so"
