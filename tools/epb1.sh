out=gpurun_out/epb1; mkdir -p $out
NBK_EXTRA_FLAGS="-DNBK_EPB8_F32=1" python -m paper_2405_11065_b200.build --force > $out/build.log 2>&1
for c in C2 C4; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --others "" --no-jacobi --no-accuracy --no-precision-study > $out/b_$c.json 2>$out/b_$c.err
done
