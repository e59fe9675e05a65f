#!/bin/bash
# r2be: loader-side phase trace of small N=1 ops (where the ~1.2k cycles before the first TMA go)
OUT=gpurun_out/r2be; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
P='MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,'
for spec in "3 conv_1x1 BN=32,sk=4,sw=0,dr=0,tm=3" "0 conv_umma BN=32,sk=4,sw=0,dr=0,tm=4" "9 conv_1x1 BN=32,sk=1,sw=0,dr=0,tm=3" "42 conv_umma BN=32,sk=4,sw=0,dr=0,tm=1"; do
  set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch 1 --variant $2 --params "${P}$3" 2>&1 | head -4 | cut -c1-400
done > $OUT/traces.log
cat $OUT/traces.log
