#!/bin/bash
# usage: tools/gpu_src.sh tag config "kernel:skip ..."  -- full captures + SASS-level source CSV
tag=$1; cfg=$2; kers=$3; out=gpurun_out/$tag; mkdir -p $out
for k in $kers; do
  name=${k%%:*}; skip=${k##*:}
  rep=/tmp/src_${name}_$cfg
  timeout 900 ncu --clock-control none --set full --import-source on -k regex:$name --launch-skip $skip -c 1 -o $rep -f \
    python tools/run_solve.py --config $cfg --precision fp32 --reps 1 --niter 3 > $out/src_$name.log 2>&1
  ncu -i $rep.ncu-rep --page source --csv --print-source sass > $out/sass_${name}_$cfg.csv 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > $out/raw_${name}_$cfg.csv 2>&1
  gzip -f $out/sass_${name}_$cfg.csv
done
