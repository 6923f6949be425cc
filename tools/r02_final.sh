#!/bin/bash
# Round-2 final evidence on one B200: smoke, full GPU suite, bench line, no-wait batch rate,
# then the k_batch launch list and one ncu --set full capture of the same build.
OUT=${1:-gpurun_out/final}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
python -m pytest tests -m gpu -q --durations=25 > $OUT/pytest.log 2>&1; echo "pytest_rc=$?" >> $OUT/pytest.log
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
python tools/nowait_batch_rate.py > $OUT/nowait_batch.json 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sharded --e2e-steps 1"
$B > $OUT/plain_batch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_batch.csv $B > $OUT/ncu_launch_batch.log 2>&1
echo "launch_rc=$?" >> $OUT/ncu_rc.txt
$B > $OUT/plain_batch2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:^k_batch$ -c 1 -o $OUT/k_batch $B > $OUT/ncu_batch.log 2>&1
echo "full_rc=$?" >> $OUT/ncu_rc.txt
bash tools/quick_single.sh $OUT
# the k_grid captures (~15 MB each) only when asked: gpurun copies back at most 64 MiB
declare -A IT=( [ontario]=500 [large]=300 [surge]=20 )
for w in ${KGRID_NCU:-}; do
  cmd="python bench.py --workload $w --iters ${IT[$w]} --steps 1 --warmup 0 --no-cpu-baseline"
  $cmd > $OUT/plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_grid -c 1 -o $OUT/k_grid_$w $cmd > $OUT/ncu_$w.log 2>&1
  echo "$w ncu rc=$?" >> $OUT/ncu_rc.txt
done
