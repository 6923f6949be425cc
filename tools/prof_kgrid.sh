#!/bin/bash
# Fresh k_grid evidence for the single-instance configs (C2/C4/C5): timings with clocks,
# then one ncu --set full capture per config of the same command (plain run first).
# usage: tools/prof_kgrid.sh TAG
set -u
TAG=${1:-r02}
OUT=gpurun_out/kgrid_$TAG
mkdir -p $OUT
for w in ontario large surge; do
  timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
# short captures: C2 500 iterations, C4 300, C5 20 (persistent kernel = one launch)
declare -A IT=( [ontario]=500 [large]=300 [surge]=20 )
for w in ontario large surge; do
  cmd="python bench.py --workload $w --iters ${IT[$w]} --steps 1 --warmup 0 --no-cpu-baseline"
  $cmd > $OUT/plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_grid -c 1 -o $OUT/k_grid_$w $cmd > $OUT/ncu_$w.log 2>&1
  echo "$w ncu rc=$?"
done
