#!/bin/bash
# r2bo: upper bound for a split-free first-layer path: timings with the A split skipped (debug bit 3, results invalid)
OUT=gpurun_out/r2bo; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
P='MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,'
for spec in "35 BN=64,sk=1,sw=0,dr=0,tm=1,pr=1" "35 BN=64,sk=1,sw=0,dr=0,tm=1" "35 BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" "33 BN=128,sk=1,sw=0,dr=0,tm=6,pr=1"; do
  set -- $spec
  for fl in 1 9 3; do
    timeout 120 python tools/trace_op.py --row $1 --batch 20 --params "${P}$2" --flags $fl 2>&1 | grep -E "^time with" | sed "s/^/row$1 $2 /"
  done
done > $OUT/times.log; cat $OUT/times.log
