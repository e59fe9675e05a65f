OUT=gpurun_out/first1
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "34 20 conv_umma BN=96,sk=1,sw=0,dr=0,tm=1" "35 20 conv_umma BN=64,sk=1,sw=0,dr=0,tm=1" "35 20 conv_umma BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" "20 20 conv_1x1 BN=96,sk=1,sw=0,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --variant $3 --params "$P,$4" >> $OUT/trace.log 2>&1
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --variant $3 --params "$P,$4" --flags 0,2,4,8 >> $OUT/ovh.log 2>&1
done
cat $OUT/ovh.log
