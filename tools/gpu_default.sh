#!/bin/bash
# The driver's round-end sequence on one GPU: gpu tests, smoke, default bench, reference arm,
# and the ncu launch list of the bench command (profiles/).
tag=${1:-d}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/smi.txt 2>&1
[ -z "$SKIP_TESTS" ] && timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
t0=$(date +%s); timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "$(( $(date +%s) - t0 )) s" > $out/bench_time.txt
[ -z "$SKIP_REF" ] && timeout 900 python bench.py --impl reference > $out/bench_reference.json 2> $out/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $out/launches_bench.csv python bench.py --steps 2 --warmup 1 --others "" --no-cpu-baseline > $out/ncu_bench.log 2>&1
