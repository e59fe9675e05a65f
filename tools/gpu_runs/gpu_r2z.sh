#!/bin/bash
# r2z: first-layer (C=3) ops: phase trace and tile options
OUT=gpurun_out/r2z; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
timeout 60 python tools/trace_op.py --row 34 --batch 20 --params "$B,BN=96,sk=1,sw=0,dr=0,tm=1" > $OUT/trace34.log 2>&1
timeout 60 python tools/trace_op.py --row 34 --batch 20 --params "$B,BN=96,sk=1,sw=0,dr=0,tm=1" --flags 3 > $OUT/trace34_hihi.log 2>&1
timeout 60 python tools/trace_op.py --row 35 --batch 20 --params "$B,BN=64,sk=1,sw=0,dr=0,tm=1" > $OUT/trace35.log 2>&1
P="BN=96,sk=1,tm=1 BN=128,sk=1,tm=1 BN=96,sk=1,tm=1,cl=3 BN=64,sk=1,tm=1,oc=2 BN=64,sk=1,tm=1,cl=3 BN=96,sk=0,tm=1 BN=192,sk=1,tm=1"
timeout 300 python tools/try_params.py --ops 34:20,33:20,35:20,34:5 --params $P > $OUT/try.log 2>&1
cat $OUT/try.log | grep -v "^ \|Traceback\|File\|torch\.\|return"
head -12 $OUT/trace34.log | cut -c1-400; grep "time" $OUT/trace34_hihi.log; head -3 $OUT/trace35.log | cut -c1-300
