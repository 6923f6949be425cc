# same-box A/B of the batched kernel: the current library against libairsched_old.so, C3 bench lines
mkdir -p gpurun_out/abb
L=paper_2002_11710_b200
cp $L/libairsched.so /tmp/lib_new.so
for round in 1 2; do
  cp /tmp/lib_new.so $L/libairsched.so
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sharded 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'new','value':d['value']}))" >> gpurun_out/abb/ab.jsonl
  cp $L/libairsched_old.so $L/libairsched.so
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sharded 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'old','value':d['value']}))" >> gpurun_out/abb/ab.jsonl
done
cp /tmp/lib_new.so $L/libairsched.so
