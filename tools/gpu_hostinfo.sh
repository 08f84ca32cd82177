#!/bin/bash
# usage: tools/gpu_hostinfo.sh out_dir -- host memory / cores / GPU of the box
out=${1:-gpurun_out}; mkdir -p $out
{ free -g; nproc; python -c "import os;print('affinity',len(os.sched_getaffinity(0)))"; grep -m1 'model name' /proc/cpuinfo; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; } > $out/hostinfo.txt 2>&1
