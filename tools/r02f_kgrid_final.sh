mkdir -p gpurun_out/r02f
python bench.py --oracle-baselines gpurun_out/r02f/oracle_baseline.jsonl > gpurun_out/r02f/oracle_baseline.log 2>&1
bash tools/quick_single.sh gpurun_out/r02f
OUT=gpurun_out/r02f
declare -A IT=( [ontario]=500 [large]=300 [surge]=20 )
for w in ontario large surge; do
  cmd="python bench.py --workload $w --iters ${IT[$w]} --steps 1 --warmup 0 --no-cpu-baseline"
  $cmd > $OUT/plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_grid -c 1 -o $OUT/k_grid_$w $cmd > $OUT/ncu_$w.log 2>&1
  echo "$w ncu rc=$?" >> $OUT/ncu_rc.txt
done
