OUT=gpurun_out/p9
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "6 1 BN=32,sk=1,sw=0,dr=0,tm=1" "40 1 BN=32,sk=8,sw=1,dr=0,tm=1" "17 1 BN=32,sk=4,sw=0,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3" --flags 0,16 >> $OUT/ovh.log 2>&1
  B2C_NO_PDL=1 timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3" --flags 0,16 | sed 's/^/NOPDL /' >> $OUT/ovh.log 2>&1
done
timeout 120 python tools/op_overhead.py --row 6 --batch 1 --variant conv_simple --params "$P" --flags 0 >> $OUT/ovh.log 2>&1
