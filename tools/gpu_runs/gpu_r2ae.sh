#!/bin/bash
OUT=gpurun_out/r2ae; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "42 20 conv_umma BN=128,sk=1,sw=0,dr=0,tm=5,pr=1" "42 20 conv_umma BN=128,sk=1,sw=0,dr=0,tm=1" "0 1 conv_umma BN=32,sk=4,sw=0,dr=0,tm=4" "6 20 conv_1x1 BN=64,sk=1,sw=0,dr=0,tm=3"; do
  set -- $spec
  timeout 60 python tools/trace_op.py --row $1 --batch $2 --variant $3 --params "$B,$4" 2>&1 | sed -n 1,3p | cut -c1-400
done > $OUT/trace.log
cat $OUT/trace.log
