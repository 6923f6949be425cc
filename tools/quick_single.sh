#!/bin/bash
# single-instance timings (TS and NS) with clock records: each config repeated until >= 1 s of timed region
# usage: tools/quick_single.sh OUTDIR [workloads...]
OUT=${1:-gpurun_out/single}
shift
WL=${@:-tiny ontario large surge}
mkdir -p $OUT
for w in $WL; do for ns in "" "--ns"; do
  timeout 300 python bench.py --workload $w $ns --steps 3 --warmup 3 --min-seconds 1.0 --no-cpu-baseline 2>>$OUT/err.log | tail -1 >> $OUT/single_configs.jsonl
done; done
