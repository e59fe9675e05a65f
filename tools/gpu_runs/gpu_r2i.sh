#!/bin/bash
# r2i: 2-SM UMMA pairs (cl=3): golden parity of every variant, then timings vs single CTAs
OUT=gpurun_out/r2i; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 420 python -m pytest tests/test_gpu_parity.py -q -x -k golden > $OUT/pytest_golden.log 2>&1; echo "exit $?" >> $OUT/pytest_golden.log
tail -15 $OUT/pytest_golden.log
P="BN=128,sk=0,tm=1 BN=128,sk=1,tm=1 BN=128,sk=1,tm=1,cl=3 BN=192,sk=1,tm=1,cl=3 BN=64,sk=1,tm=1,cl=3 BN=128,sk=2,tm=1,cl=3 BN=192,sk=1,tm=1 BN=128,sk=1,tm=1,cl=2"
timeout 300 python tools/try_params.py --ops 42:20,41:20,40:20,39:20,38:20 --params $P > $OUT/try.log 2>&1
cat $OUT/try.log
P4="BN=128,sk=1,tm=4 BN=192,sk=1,tm=4 BN=128,sk=1,tm=4,cl=3 BN=192,sk=1,tm=4,cl=3 BN=64,sk=1,tm=4,cl=3"
timeout 300 python tools/try_params.py --ops 41:20,39:20,31:20 --params $P4 > $OUT/try4.log 2>&1
cat $OUT/try4.log
P3="BN=64,sk=1,tm=3 BN=128,sk=1,tm=3 BN=64,sk=1,tm=3,cl=3 BN=128,sk=1,tm=3,cl=3 BN=192,sk=1,tm=3,cl=3"
timeout 300 python tools/try_params.py --ops 6:20,20:20,27:20,24:20 --params $P3 > $OUT/try3.log 2>&1
cat $OUT/try3.log
B="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
{
python tools/trace_op.py --row 6 --batch 20 --variant conv_1x1 --params "$B,BN=64,sk=1,sw=0,dr=0,tm=3"
python tools/trace_op.py --row 3 --batch 20 --variant conv_1x1 --params "$B,BN=64,sk=1,sw=0,dr=0,tm=3"
python tools/trace_op.py --row 0 --batch 1 --params "$B,BN=32,sk=4,sw=0,dr=0,tm=4"
python tools/trace_op.py --row 3 --batch 1 --variant conv_1x1 --params "$B,BN=32,sk=4,sw=0,dr=0,tm=3"
python tools/trace_op.py --row 26 --batch 20 --params "$B,BN=64,sk=1,sw=0,dr=0,tm=1"
} > $OUT/trace.log 2>&1
cat $OUT/trace.log
