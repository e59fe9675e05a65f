OUT=gpurun_out/p11
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
timeout 120 python tools/trace_op.py --row 40 --batch 1 --params "$P,BN=32,sk=8,sw=1,dr=0,tm=1" --flags 1 2>&1 | grep -v "rep0" >> $OUT/trace.log
timeout 120 python tools/trace_op.py --row 40 --batch 1 --params "$P,BN=32,sk=8,sw=1,dr=0,tm=1" --flags 3 2>&1 | grep -v "rep0" >> $OUT/trace.log
timeout 120 python tools/trace_op.py --row 40 --batch 1 --params "$P,BN=32,sk=8,sw=1,dr=0,tm=1" --flags 7 2>&1 | grep -v "rep0" >> $OUT/trace.log
