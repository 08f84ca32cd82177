#!/bin/bash
# K_B warp-stream bring-up: parity tests, A/B against the block-barrier K_B and launch variants, ncu of K_B
out=gpurun_out/kb2; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pcg.py tests/test_gpu_single.py tests/test_gpu_multirank.py tests/test_gpu_dssum_stage.py -x -q > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
tail -3 $out/pytest.log
tools/ab_envs.sh kb2/ab "C5 C4" "NBK_LIB=build_ab/libkbold.so" "NBK_LIB=build_ab/libkbw4.so" "NBK_DSSUM_TILE_NODES=2048" "NBK_DSSUM_TILE_NODES=128"
tools/gpu_kfull.sh kb2/fullB C5 fp32 k_dssum 1
