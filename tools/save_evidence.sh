#!/bin/bash
# usage: tools/save_evidence.sh src_tag "note" -- copy a gpu_round_end.sh run (gpurun_out/<tag>) into
# profiles/r02 and regenerate profiles/r02_ncu.md + profiles/ncu_summary.json from its raw pages
src=gpurun_out/$1; note=$2; dst=profiles/r02
for f in bench_default.json bench_reference.json launches_bench.csv pytest_gpu.log smoke.log; do
  [ -f $src/$f ] && cp $src/$f $dst/$f
done
mkdir -p $dst/ncu_raw
cp $src/raw_*.csv $src/launches_C*.csv $dst/ncu_raw/ 2>/dev/null
reps=""
for c in C5 C4 C3; do for p in fp32 fp64; do for k in k_ax k_dssum k_vec; do
  f=$dst/ncu_raw/raw_${k}_${c}_${p}.csv; [ -f $f ] && reps="$reps --rep $c:$p:$f"
done; done; done
python tools/ncu_summary.py --round r02 --fresh --note "$note" $reps \
  --launches C5:$dst/ncu_raw/launches_C5.csv --launches bench:$dst/launches_bench.csv
