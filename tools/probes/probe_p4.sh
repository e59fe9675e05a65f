OUT=gpurun_out/p4
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "42 20 BN=128,sk=1,sw=0,dr=0,tm=1" "34 20 BN=96,sk=1,sw=0,dr=0,tm=1" "41 20 BN=192,sk=1,sw=0,dr=0,tm=1" "20 20 BN=96,sk=1,sw=0,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3" --flags 16,18,20,22 >> $OUT/ovh.log 2>&1
done
