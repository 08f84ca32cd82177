#!/bin/bash
# usage: tools/gpu_prof.sh tag config [kernels]  -- launch list + full captures (FP32, steady state)
# Exports raw/details CSV on the box; keeps compressed reports only while under the 64 MiB cap.
tag=${1:-p}; cfg=${2:-C4}; kers=${3:-"k_ax:1 k_dssum:1 k_vec:3"}; out=gpurun_out/$tag; mkdir -p $out
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $out/launches_$cfg.csv python tools/run_solve.py --config $cfg --precision fp32,fp64 --reps 1 --niter 4 > $out/launch.log 2>&1
for k in $kers; do
  name=${k%%:*}; skip=${k##*:}
  rep=/tmp/full_${name}_$cfg
  timeout 900 $NCU --set full --import-source on -k regex:$name --launch-skip $skip -c 1 -o $rep -f \
    python tools/run_solve.py --config $cfg --precision fp32 --reps 1 --niter 3 > $out/full_$name.log 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > $out/raw_${name}_$cfg.csv 2>&1
  ncu -i $rep.ncu-rep --page details --csv > $out/details_${name}_$cfg.csv 2>&1
  ncu -i $rep.ncu-rep --page source --csv > $out/source_${name}_$cfg.csv 2>&1
  gzip -f $out/source_${name}_$cfg.csv
  ls -la $rep.ncu-rep >> $out/sizes.txt
done
du -sh $out >> $out/sizes.txt
