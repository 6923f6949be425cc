mkdir -p gpurun_out/r02o
L=paper_2002_11710_b200
cp $L/libairsched.so /tmp/lib_a.so
python tools/kgrid_quick.py A > gpurun_out/r02o/ab.jsonl 2>&1
cp $L/libairsched_noph.so $L/libairsched.so
python tools/kgrid_quick.py B_nophase >> gpurun_out/r02o/ab.jsonl 2>&1
cp /tmp/lib_a.so $L/libairsched.so
python tools/kgrid_quick.py A2 >> gpurun_out/r02o/ab.jsonl 2>&1
cp $L/libairsched_noph.so $L/libairsched.so
python tools/kgrid_quick.py B2_nophase >> gpurun_out/r02o/ab.jsonl 2>&1
