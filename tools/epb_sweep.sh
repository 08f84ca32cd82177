out=gpurun_out/stg; mkdir -p $out
for v in 16 8; do
  NBK_EXTRA_FLAGS="-DNBK_STAGE_G_MAXN=$v" python -m paper_2405_11065_b200.build --force > $out/build_$v.log 2>&1
  grep -A2 "k_axIfLi12ELi1E\|k_axIfLi10ELi1E\|k_axIdLi12ELi1E\|k_axIdLi10ELi1E" paper_2405_11065_b200/csrc/nbk_capi.ptxas.log | grep -E "registers|spill" >> $out/build_$v.log
  for c in C3 C5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --others "" --no-jacobi --no-accuracy > $out/b_${v}_$c.json 2>/dev/null
  done
done
