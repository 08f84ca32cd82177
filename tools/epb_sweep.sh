out=gpurun_out/epb; mkdir -p $out
for v in "3 2" "2 1" "2 2" "3 1"; do
  set -- $v
  NBK_EXTRA_FLAGS="-DNBK_EPB8_F32=$1 -DNBK_EPB8_F64=$2" python -m paper_2405_11065_b200.build --force > /dev/null 2>&1
  for c in C2 C4; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --others "" --no-jacobi --no-accuracy > $out/b_${1}_${2}_$c.json 2>/dev/null
  done
done
