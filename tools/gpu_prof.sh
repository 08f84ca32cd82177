#!/bin/bash
# usage: tools/gpu_prof.sh tag config [kernels]  -- launch list + ncu --set full captures of the
# steady-state K_A / K_B / K_C launches (FP32 and FP64 solver).  Exports raw/details/source CSV on
# the box (reports stay there: the merge-back cap is 64 MiB).
tag=${1:-p}; cfg=${2:-C4}; kers=${3:-"k_ax:1 k_dssum:1 k_vec:3"}; out=gpurun_out/$tag; mkdir -p $out
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $out/launches_$cfg.csv python tools/run_solve.py --config $cfg --precision fp32,fp64 --reps 1 --niter 4 > $out/launch.log 2>&1
for prec in fp32 fp64; do
for k in $kers; do
  name=${k%%:*}; skip=${k##*:}
  rep=/tmp/full_${name}_${cfg}_$prec
  timeout 900 $NCU --set full --import-source on -k regex:$name --launch-skip $skip -c 1 -o $rep -f \
    python tools/run_solve.py --config $cfg --precision $prec --reps 1 --niter 3 > $out/full_${name}_$prec.log 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > $out/raw_${name}_${cfg}_$prec.csv 2>&1
  ncu -i $rep.ncu-rep --page details --csv > $out/details_${name}_${cfg}_$prec.csv 2>&1
  ls -la $rep.ncu-rep >> $out/sizes.txt
done
done
