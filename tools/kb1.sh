# One ncu --set full capture of k_batch on the bench's C3 launch (after a plain run of the same command).
# usage: tools/kb1.sh OUTDIR
OUT=gpurun_out/${1:-kb1}; mkdir -p $OUT
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sharded --e2e-steps 1"
$B > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_batch$ -c 1 -o $OUT/k_batch $B > $OUT/ncu.log 2>&1
echo "rc=$?"
