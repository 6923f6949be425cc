#!/bin/bash
# Round-2 evidence: launch lists + one ncu --set full capture per dominant kernel of the same build.
#   k_batch  : bench.py default workload (C3), 1 step
#   k_grid   : C2 (500 it), C4 (300 it), C5 (20 it) single-instance runs
# Every ncu command is preceded by the same command without ncu (&&).
set -u
OUT=${1:-gpurun_out/prof_r02}
mkdir -p $OUT
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sharded --e2e-steps 1"
$B > $OUT/plain_batch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_batch.csv $B > $OUT/ncu_launch_batch.log 2>&1
$B > $OUT/plain_batch2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:^k_batch$ -c 1 -o $OUT/k_batch $B > $OUT/ncu_batch.log 2>&1
declare -A IT=( [ontario]=500 [large]=300 [surge]=20 )
for w in ontario large surge; do
  cmd="python bench.py --workload $w --iters ${IT[$w]} --steps 1 --warmup 0 --no-cpu-baseline"
  $cmd > $OUT/plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_grid -c 1 -o $OUT/k_grid_$w $cmd > $OUT/ncu_$w.log 2>&1
  echo "$w ncu rc=$?"
done
