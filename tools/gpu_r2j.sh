#!/bin/bash
out=gpurun_out/r2j; mkdir -p $out
NBK_LIB=build_ab/libnbk_g2.so timeout 600 python -m pytest tests -m gpu -x -q -k "dssum or c2_history or pcg_c2 or small_meshes or vprec_solver_bitwise or mca_samples" > $out/pytest_g2.log 2>&1; echo "rc=$?" >> $out/pytest_g2.log
B="--steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others '' --no-accuracy --no-jacobi --energy-reps 1"
for rep in 1 2; do
for c in C5 C4; do
  for tn in 1024 512 2048; do
    NBK_DSSUM_TILE_NODES=$tn timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/A_t${tn}_${c}_$rep.json 2> $out/A_t${tn}_${c}_$rep.err
    NBK_LIB=build_ab/libnbk_g2.so NBK_DSSUM_TILE_NODES=$tn timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/G2_t${tn}_${c}_$rep.json 2> $out/G2_t${tn}_${c}_$rep.err
    NBK_LIB=build_ab/libnbk_kb6.so NBK_DSSUM_TILE_NODES=$tn timeout 600 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-precision-study --convergence 0 --others "" --no-accuracy --no-jacobi --energy-reps 1 > $out/KB6_t${tn}_${c}_$rep.json 2> $out/KB6_t${tn}_${c}_$rep.err
  done
done
done
