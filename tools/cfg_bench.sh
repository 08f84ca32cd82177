# usage: tools/cfg_bench.sh tag [configs] -- GPU tests + per-config bench lines
tag=${1:-cb}; cfgs=${2:-"C2 C4 C3 C5"}; out=gpurun_out/$tag; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
for c in $cfgs; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --others "" --no-jacobi --no-accuracy --no-precision-study > $out/b_$c.json 2>$out/b_$c.err
done
