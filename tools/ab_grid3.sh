# same-box A/B/C of the whole-GPU kernel: current library (default and with the options in $1),
# and libairsched_old.so (tools/kgrid_quick.py)
mkdir -p gpurun_out/abg
L=paper_2002_11710_b200
cp $L/libairsched.so /tmp/lib_new.so
for round in 1 2; do
  cp /tmp/lib_new.so $L/libairsched.so; python tools/kgrid_quick.py new_$round >> gpurun_out/abg/ab.jsonl 2>&1
  python tools/kgrid_quick.py newopt_$round $1 >> gpurun_out/abg/ab.jsonl 2>&1
  cp $L/libairsched_old.so $L/libairsched.so; python tools/kgrid_quick.py old_$round >> gpurun_out/abg/ab.jsonl 2>&1
done
cp /tmp/lib_new.so $L/libairsched.so
