#!/bin/bash
# r2aa: is the split (A -> TMEM) role the bottleneck?  timings with the A split skipped (debug bit 3, results invalid)
OUT=gpurun_out/r2aa; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
{
for spec in "34 20 conv_umma BN=96,sk=1,sw=0,dr=0,tm=1" "35 20 conv_umma BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" "6 20 conv_1x1 BN=64,sk=1,sw=0,dr=0,tm=3" \
            "27 20 conv_1x1 BN=64,sk=1,sw=0,dr=0,tm=2,oc=2" "42 20 conv_umma BN=128,sk=0,sw=0,dr=0,tm=1,cl=3" "40 20 conv_umma BN=128,sk=1,sw=0,dr=0,tm=1,cl=3" \
            "38 1 conv_umma BN=32,sk=8,sw=0,dr=0,tm=1,oc=2" "42 5 conv_umma BN=128,sk=1,sw=0,dr=0,tm=1,cl=3" "25 20 conv_fc BN=32,sk=8,sw=1,dr=0,tm=1,oc=2"; do
  set -- $spec
  for fl in 0 2 8 10; do
    timeout 60 python tools/op_overhead.py --row $1 --batch $2 --variant $3 --params "$B,$4" --flags $fl --k 20 2>&1 | tail -1
  done
done
} > $OUT/split_cost.log 2>&1
cat $OUT/split_cost.log
