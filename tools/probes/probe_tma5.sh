OUT=gpurun_out/tma5
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "17 1 BN=32,sk=1,sw=0" "42 20 BN=128,sk=1,sw=0"; do set -- $spec
  for fl in 1 9; do
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" --flags $fl 2>&1 | grep -v "rep0" >> $OUT/trace.log
  done
done
