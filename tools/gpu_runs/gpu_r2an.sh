#!/bin/bash
# r2an: SPLIT2 (second split group, OCC 1, BN <= 64) + FUSED (OCC 1): fc6/fc7 tile options, small-op retime, traces
OUT=gpurun_out/r2an; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $OUT/pytest_parity.log 2>&1; tail -2 $OUT/pytest_parity.log
P='MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,'
timeout 600 python tools/try_params.py --ops 25:20,25:5,13:20,13:5 --params \
  "conv_fc:BN=32,sk=8,sw=1,dr=0,tm=1,oc=2" "conv_fc:BN=32,sk=8,sw=1,dr=0,tm=1" "conv_fc:BN=32,sk=9,sw=1,dr=0,tm=1" \
  "conv_fc:BN=32,sk=0,sw=1,dr=0,tm=1" "conv_fc:BN=32,sk=4,sw=1,dr=0,tm=1" "conv_fc:BN=32,sk=16,sw=1,dr=0,tm=1" \
  "conv_fc:BN=32,sk=16,sw=1,dr=0,tm=1,oc=2" > $OUT/fc_try.log 2>&1; cat $OUT/fc_try.log
timeout 300 python tools/trace_op.py --row 25 --batch 20 --variant conv_fc --params "${P}BN=32,sk=8,sw=1,dr=0,tm=1" > $OUT/trace_fc6_occ1.log 2>&1
timeout 300 python tools/trace_op.py --row 0 --batch 1 --params "${P}BN=32,sk=4,sw=0,dr=0,tm=4" > $OUT/trace_row0.log 2>&1
timeout 900 python tools/db_retime.py --only-bn 32,64 --csv $OUT/retime_fp32.csv > $OUT/retime_fp32.log 2>&1; tail -1 $OUT/retime_fp32.log
grep -c FAIL $OUT/retime_fp32.log
