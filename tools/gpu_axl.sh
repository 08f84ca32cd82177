#!/bin/bash
# usage: tools/gpu_axl.sh tag "variant libs" "configs" [pytest files]  -- K_A line-owner bring-up:
# parity tests, same-box A/B bench against variant builds, ncu wavefront / DRAM metrics of K_A at C5.
tag=${1:-axl}; libs=$2; cfgs=${3:-"C5"}; tests=${4:-"tests/test_gpu_parity.py tests/test_gpu_pcg.py tests/test_gpu_single.py tests/test_gpu_multirank.py"}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 1500 python -m pytest $tests -x -q > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
tail -3 $out/pytest.log
[ -n "$libs" ] && tools/ab_lib.sh $tag/ab "$libs" "$cfgs"
python tools/ab_show.py $out/ab 2>/dev/null | tail -20
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
for c in $cfgs; do
timeout 600 ncu --clock-control none --metrics $M -k regex:k_ax --launch-skip 1 -c 2 --csv --log-file $out/ncu_kax_$c.csv \
  python tools/run_solve.py --config $c --precision fp32,fp64 --reps 1 --niter 3 > $out/ncu_$c.log 2>&1
done
