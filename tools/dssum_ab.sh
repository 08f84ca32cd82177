# A/B of K_B nodes-per-thread (H) and FP32 min blocks: C2 and C4 FP32/FP64
out=gpurun_out/dsab; mkdir -p $out
for v in "2 4" "4 3" "4 4" "3 4"; do
  set -- $v
  NBK_EXTRA_FLAGS="-DNBK_DSSUM_H=$1 -DNBK_DSSUM_MINB32=$2" python -m paper_2405_11065_b200.build --force > $out/build_$1_$2.log 2>&1
  grep -A2 "k_dssumIfLb1ELi0E\|k_dssumIdLb1ELi0E" paper_2405_11065_b200/csrc/nbk_capi.ptxas.log | grep -E "registers|spill" >> $out/build_$1_$2.log
  for c in C2 C4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --others "" --no-jacobi --no-accuracy --no-precision-study > $out/b_$1_$2_$c.json 2>$out/b_$1_$2_$c.err
  done
done
