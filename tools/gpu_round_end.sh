#!/bin/bash
# usage: tools/gpu_round_end.sh tag -- full -m gpu suite, smoke(), then tools/gpu_final.sh (bench line,
# reference arm, ncu launch list and full captures)
tag=${1:-end}; out=gpurun_out/$tag; mkdir -p $out
( time timeout 2400 python -m pytest tests -m gpu -q --durations=10 ) > $out/pytest_gpu.log 2>&1; echo "rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "rc=$?" >> $out/smoke.log
( time tools/gpu_final.sh $tag ) > $out/final_time.log 2>&1
