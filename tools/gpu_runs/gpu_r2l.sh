#!/bin/bash
# r2l: pair-mode timing after the relaxed drain arrive; pair trace; launch-floor decomposition of small ops
OUT=gpurun_out/r2l; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k golden > $OUT/pytest_golden.log 2>&1; echo "exit $?" >> $OUT/pytest_golden.log
tail -2 $OUT/pytest_golden.log
P="BN=128,sk=0,tm=1 BN=128,sk=1,tm=1 BN=128,sk=1,tm=1,cl=3 BN=192,sk=1,tm=1,cl=3 BN=128,sk=2,tm=1,cl=3"
timeout 300 python tools/try_params.py --ops 42:20,40:20,39:20 --params $P > $OUT/try.log 2>&1
cat $OUT/try.log
B="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
{
timeout 60 python tools/trace_op.py --row 42 --batch 20 --params "$B,BN=128,sk=1,sw=0,dr=0,tm=1,cl=3"
timeout 60 python tools/trace_op.py --row 42 --batch 20 --params "$B,BN=128,sk=1,sw=0,dr=0,tm=1"
} > $OUT/trace.log 2>&1
{
timeout 60 python tools/launch_floor.py --row 3 --batch 1 --variant conv_1x1 --params "BN=32,sk=4,sw=0,dr=0,tm=3"
timeout 60 python tools/launch_floor.py --row 3 --batch 1 --variant conv_1x1 --params "BN=32,sk=1,sw=0,dr=0,tm=3"
timeout 60 python tools/launch_floor.py --row 6 --batch 20 --variant conv_1x1 --params "BN=64,sk=1,sw=0,dr=0,tm=3"
timeout 60 python tools/launch_floor.py --row 0 --batch 1 --params "BN=32,sk=4,sw=0,dr=0,tm=4"
timeout 60 python tools/launch_floor.py --row 42 --batch 1 --params "BN=32,sk=4,sw=0,dr=0,tm=1"
} > $OUT/floor.log 2>&1
cat $OUT/floor.log
