mkdir -p gpurun_out/r02p
L=paper_2002_11710_b200
cp $L/libairsched.so /tmp/lib_a.so
for round in 1 2; do
  cp /tmp/lib_a.so $L/libairsched.so; python tools/kgrid_quick.py W24_$round >> gpurun_out/r02p/ab.jsonl 2>&1
  cp $L/libairsched_w20.so $L/libairsched.so; python tools/kgrid_quick.py W20_$round >> gpurun_out/r02p/ab.jsonl 2>&1
  cp $L/libairsched_w16.so $L/libairsched.so; python tools/kgrid_quick.py W16_$round >> gpurun_out/r02p/ab.jsonl 2>&1
done
cp /tmp/lib_a.so $L/libairsched.so
