#!/bin/bash
# usage: tools/gpu_kfull.sh tag config prec kernel_regex [skip]  -- one ncu --set full capture of a
# kernel with raw / details / source (SASS + CUDA, per-line stalls) pages exported as CSV.
tag=$1; cfg=$2; prec=$3; k=$4; skip=${5:-1}; out=gpurun_out/$tag; mkdir -p $out
rep=/tmp/full_${cfg}_$prec
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip $skip -c 1 -o $rep -f \
  python tools/run_solve.py --config $cfg --precision $prec --reps 1 --niter 3 > $out/full_${cfg}_$prec.log 2>&1
ncu -i $rep.ncu-rep --page raw --csv > $out/raw_${cfg}_$prec.csv 2>&1
ncu -i $rep.ncu-rep --page details --csv > $out/details_${cfg}_$prec.csv 2>&1
ncu -i $rep.ncu-rep --page source --csv --print-source sass > $out/sass_${cfg}_$prec.csv 2>&1
ncu -i $rep.ncu-rep --page source --csv --print-source cuda > $out/cuda_${cfg}_$prec.csv 2>&1
ls -la $out
