#!/bin/bash
# single-instance timings (TS and NS) with clock records: each step repeated until >= 1 s of timed region
OUT=${1:-gpurun_out/single}
mkdir -p $OUT
for w in tiny ontario large surge; do for ns in "" "--ns"; do
  timeout 300 python bench.py --workload $w $ns --steps 3 --warmup 3 --min-seconds 1.0 --no-cpu-baseline 2>>$OUT/err.log | tail -1 >> $OUT/single_configs.jsonl
done; done
