out=gpurun_out/minb; mkdir -p $out
for v in "1 4" "4 4" "6 6" "5 5"; do
  set -- $v
  NBK_EXTRA_FLAGS="-DNBK_VEC_MINB=$1 -DNBK_DSSUM_MINB32=$2" python -m paper_2405_11065_b200.build --force > /dev/null 2>&1
  grep -A2 "k_vecIfLi8ELi1E\|k_dssumIfLb1" paper_2405_11065_b200/csrc/nbk_capi.ptxas.log | grep -E "registers|spill" > $out/regs_$1_$2.txt
  for c in C2 C4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --others "" --no-jacobi --no-accuracy > $out/b_$1_$2_$c.json 2>/dev/null
  done
done
