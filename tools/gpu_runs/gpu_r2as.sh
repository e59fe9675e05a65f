#!/bin/bash
# r2as: phase traces of the first-layer kernels (what paces a K block: TMA, split or MMA)
OUT=gpurun_out/r2as; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
P='MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,'
for spec in "34 BN=96,sk=1,sw=0,dr=0,tm=6,cl=3" "34 BN=96,sk=1,sw=0,dr=0,tm=1,cl=3" "34 BN=96,sk=1,sw=0,dr=0,tm=1" "35 BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" "35 BN=64,sk=1,sw=0,dr=0,tm=1" "42 BN=128,sk=1,sw=0,dr=0,tm=1"; do
  set -- $spec
  for fl in 1 3 5 9; do
    timeout 120 python tools/trace_op.py --row $1 --batch 20 --params "${P}$2" --flags $fl 2>&1 | grep -E "^---|time with" | head -2
  done
done > $OUT/traces_summary.log
cat $OUT/traces_summary.log
for spec in "34 BN=96,sk=1,sw=0,dr=0,tm=1" "35 BN=64,sk=1,sw=0,dr=0,tm=1"; do
  set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch 20 --params "${P}$2" --flags 1 > $OUT/trace_r$1.log 2>&1
done
