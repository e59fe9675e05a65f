OUT=gpurun_out/p5
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "20 20 BN=96,sk=1,sw=0,dr=0,tm=1" "42 20 BN=128,sk=1,sw=0,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --params "$P,$3" --flags 1 2>&1 | grep -v "rep0" >> $OUT/trace.log
done
