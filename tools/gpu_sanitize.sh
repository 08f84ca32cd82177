#!/bin/bash
# usage: tools/gpu_sanitize.sh tag -- compute-sanitizer memcheck / racecheck / synccheck / initcheck
tag=${1:-san}; out=gpurun_out/$tag; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_run.py > $out/sanitize_$tool.log 2>&1
  echo "exit=$?" >> $out/sanitize_$tool.log
done
