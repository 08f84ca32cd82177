#!/bin/bash
# usage: tools/gpu_final.sh tag -- default bench line, reference arm, ncu launch list of the bench
# command, ncu --set full captures of K_A / K_B / K_C at C5 (+ K_A at C3, C4)
tag=${1:-final}; out=gpurun_out/$tag; mkdir -p $out
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $out/bench_reference.json 2> $out/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv \
  --log-file $out/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-fp64 --no-cpu-baseline \
  --no-precision-study --no-accuracy --no-jacobi --others "" --prof-steps 1 --energy-reps 0 > $out/launches_bench.log 2>&1
tools/gpu_prof.sh $tag C5 "k_ax:1 k_dssum:1 k_vec:3"
tools/gpu_prof.sh $tag C3 "k_ax:1 k_dssum:1 k_vec:3"
tools/gpu_prof.sh $tag C4 "k_ax:1 k_dssum:1 k_vec:3"
