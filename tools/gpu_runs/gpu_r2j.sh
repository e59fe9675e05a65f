#!/bin/bash
# r2j: phase traces of the N=20 1x1 / small k x k ops and the N=1 split-K ops (where the per-op fixed cost goes)
OUT=gpurun_out/r2j; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
{
python tools/trace_op.py --row 6 --batch 20 --variant conv_1x1 --params "$B,BN=64,sk=1,sw=0,dr=0,tm=3"
python tools/trace_op.py --row 3 --batch 20 --variant conv_1x1 --params "$B,BN=64,sk=1,sw=0,dr=0,tm=3"
python tools/trace_op.py --row 0 --batch 1 --params "$B,BN=32,sk=4,sw=0,dr=0,tm=4"
python tools/trace_op.py --row 3 --batch 1 --variant conv_1x1 --params "$B,BN=32,sk=4,sw=0,dr=0,tm=3"
python tools/trace_op.py --row 26 --batch 20 --params "$B,BN=64,sk=1,sw=0,dr=0,tm=1"
} > $OUT/trace.log 2>&1
cat $OUT/trace.log
