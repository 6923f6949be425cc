# One ncu --set full capture of k_grid on a single-instance config (after a plain run of the same command).
# usage: tools/ks1.sh OUTDIR [WORKLOAD] [ITERS]
set -u
OUT=gpurun_out/${1:-ks1}; mkdir -p $OUT
W=${2:-surge}; IT=${3:-20}
cmd="python bench.py --workload $W --iters $IT --steps 1 --warmup 0 --no-cpu-baseline"
$cmd > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_grid -c 1 -o $OUT/k_grid_$W $cmd > $OUT/ncu.log 2>&1
echo "rc=$?"
