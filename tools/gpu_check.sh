#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench lines, ncu launch list.
# usage: tools/gpu_check.sh [tag]
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
for c in C2 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $out/bench_$c.json 2> $out/bench_$c.err
done
timeout 300 python bench.py > $out/bench_default.json 2> $out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 > $out/ncu_launch.log 2>&1
