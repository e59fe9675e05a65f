#!/bin/bash
OUT=gpurun_out/r2ad; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
timeout 60 python tools/trace_op.py --row 42 --batch 20 --params "$B,BN=128,sk=1,sw=0,dr=0,tm=5,pr=1" > $OUT/trace42_ss.log 2>&1
timeout 60 python tools/trace_op.py --row 40 --batch 20 --params "$B,BN=128,sk=1,sw=0,dr=0,tm=5,pr=1" > $OUT/trace40_ss.log 2>&1
timeout 60 python tools/op_overhead.py --row 42 --batch 20 --params "$B,BN=128,sk=1,sw=0,dr=0,tm=5,pr=1" --flags 0,16 --k 20 > $OUT/ovh.log 2>&1
cat $OUT/trace42_ss.log | head -12 | cut -c1-420; cat $OUT/ovh.log
