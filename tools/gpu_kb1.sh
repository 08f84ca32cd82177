set -x
NBK_LIB=build_ab/libkb128.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dssum_stage.py -x -q > gpurun_out/kb1_pytest.log 2>&1; echo rc=$? >> gpurun_out/kb1_pytest.log
tools/ab_envs.sh kb1 "C5 C4" "NBK_DSSUM_TILE_NODES=256" "NBK_LIB=build_ab/libkb128.so" "NBK_LIB=build_ab/libkb128.so NBK_DSSUM_TILE_NODES=256" "NBK_LIB=build_ab/libkb128.so NBK_DSSUM_TILE_NODES=128"
tools/gpu_kfull.sh kb1/fullA C5 fp32 k_axl 1
tools/gpu_kfull.sh kb1/fullB C5 fp32 k_dssum 1
