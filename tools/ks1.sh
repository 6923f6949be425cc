set -u
OUT=gpurun_out/${1:-ks1}; mkdir -p $OUT
cmd="python bench.py --workload surge --iters 20 --steps 1 --warmup 0 --no-cpu-baseline"
$cmd > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_grid -c 1 -o $OUT/k_grid_surge $cmd > $OUT/ncu.log 2>&1
echo "rc=$?"
