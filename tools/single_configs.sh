for w in tiny ontario large surge; do for ns in "" "--ns"; do timeout 300 python bench.py --workload $w $ns --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1; done; done
