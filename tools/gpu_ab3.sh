#!/bin/bash
# A/B of the padded transpose-chain layout (K_A) and the K_B segment-offset prefetch
out=gpurun_out/ab3; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pcg.py tests/test_gpu_single.py tests/test_gpu_multirank.py tests/test_gpu_dssum_stage.py -x -q > $out/pytest.log 2>&1; echo rc=$? >> $out/pytest.log
tail -3 $out/pytest.log
tools/ab_envs.sh ab3/ab "C5 C4 C3" "NBK_LIB=build_ab/libnopad.so" "NBK_LIB=build_ab/libnopf.so"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum
timeout 600 ncu --clock-control none --metrics $M -k regex:"k_ax|k_dssum" --launch-skip 2 -c 4 --csv --log-file $out/ncu_C5.csv \
  python tools/run_solve.py --config C5 --precision fp32 --reps 1 --niter 4 > $out/ncu_C5.log 2>&1
