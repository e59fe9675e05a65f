#!/bin/bash
# r2ab: the empty-pipeline floor -- phase traces with the split and 2/3 of the MMAs removed (debug flags, results invalid)
OUT=gpurun_out/r2ab; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for fl in 1 11; do
timeout 60 python tools/trace_op.py --row 42 --batch 20 --params "$B,BN=128,sk=1,sw=0,dr=0,tm=1" --flags $fl > $OUT/trace42_f$fl.log 2>&1
timeout 60 python tools/trace_op.py --row 42 --batch 20 --params "$B,BN=128,sk=1,sw=0,dr=0,tm=4" --flags $fl > $OUT/trace42tm4_f$fl.log 2>&1
timeout 60 python tools/trace_op.py --row 34 --batch 20 --params "$B,BN=96,sk=1,sw=0,dr=0,tm=1" --flags $fl > $OUT/trace34_f$fl.log 2>&1
done
for f in $OUT/trace*.log; do echo "== $f"; sed -n 2,4p $f | cut -c1-330; grep "^time" $f; done
