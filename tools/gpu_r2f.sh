mkdir -p gpurun_out/r2f
timeout 600 python -m pytest tests -m gpu -x -q -k "accum32 or test_gpu_api or single_solver" > gpurun_out/r2f/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2f/pytest.log
tools/ab_lib.sh r2f "build_ab/libnbk_presl.so" "C5 C3"
tools/gpu_prof.sh r2f C5 "k_ax:1 k_dssum:1 k_vec:3"
