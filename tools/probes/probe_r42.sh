OUT=gpurun_out/r42
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "42 20 conv_umma BN=128,sk=0,sw=0,dr=0,tm=1" "42 20 conv_umma BN=192,sk=0,sw=0,dr=0,tm=1" "41 20 conv_umma BN=192,sk=1,sw=0,dr=0,tm=1" "40 20 conv_umma BN=128,sk=0,sw=0,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --variant $3 --params "$P,$4" --flags 0,16,2,18 >> $OUT/ovh.log 2>&1
done
timeout 120 python tools/trace_op.py --row 42 --batch 20 --variant conv_umma --params "$P,BN=128,sk=0,sw=0,dr=0,tm=1" > $OUT/trace.log 2>&1
cat $OUT/ovh.log
