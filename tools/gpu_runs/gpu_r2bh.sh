#!/bin/bash
# r2bh: where the pixel loader's time goes between griddepcontrol.wait and its first TMA (trace)
OUT=gpurun_out/r2bh; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
P='MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,'
for spec in "3 conv_1x1 BN=32,sk=4,sw=0,dr=0,tm=3" "0 conv_umma BN=32,sk=4,sw=0,dr=0,tm=4"; do
  set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch 1 --variant $2 --params "${P}$3" 2>&1 | head -8 | cut -c1-320
done > $OUT/traces.log; cat $OUT/traces.log
