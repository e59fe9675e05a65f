OUT=gpurun_out/p12
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
timeout 120 python tools/trace_op.py --row 25 --batch 20 --variant conv_fc --params "$P,BN=32,sk=4,sw=1,dr=0,tm=1" --flags 1 2>&1 | grep -v "rep0" >> $OUT/trace.log
timeout 120 python tools/trace_op.py --row 25 --batch 20 --variant conv_fc --params "$P,BN=32,sk=4,sw=1,dr=0,tm=1" --flags 7 2>&1 | grep -v "rep0" >> $OUT/trace.log
for pr in "BN=32,sk=4,sw=1" "BN=32,sk=2,sw=1" "BN=32,sk=8,sw=1" "BN=64,sk=4,sw=1"; do
timeout 120 python tools/op_overhead.py --row 25 --batch 20 --variant conv_fc --params "$P,$pr,dr=0,tm=1" --flags 0 >> $OUT/ovh.log 2>&1
done
