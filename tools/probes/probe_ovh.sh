OUT=gpurun_out/ovh1
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "6 1 BN=32,sk=1,sw=0" "17 1 BN=32,sk=1,sw=0" "17 1 BN=32,sk=4,sw=0" "0 1 BN=32,sk=1,sw=0" "42 20 BN=128,sk=1,sw=0"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" --flags 0,16,18,22 >> $OUT/ovh.log 2>&1
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3,dr=0" --flags 0 >> $OUT/ovh.log 2>&1
done
timeout 120 python tools/op_overhead.py --row 6 --batch 1 --variant conv_simple --params "$P" --flags 0 >> $OUT/ovh.log 2>&1
timeout 120 python tools/op_overhead.py --row 0 --batch 1 --variant conv_tiled --params "MNt=4:4,MNb=16:16,Kb=8,vw=4,lf=1,li=1" --flags 0 >> $OUT/ovh.log 2>&1
