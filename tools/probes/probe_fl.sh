OUT=gpurun_out/fl1
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "35 20 BN=64,sk=1,sw=0,dr=0,tm=1" "35 20 BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" "35 20 BN=32,sk=1,sw=0,dr=0,tm=1,oc=2" "35 20 BN=64,sk=0,sw=0,dr=0,tm=1" "34 20 BN=96,sk=1,sw=0,dr=0,tm=1" "34 20 BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" "34 20 BN=96,sk=0,sw=0,dr=0,tm=1" "34 20 BN=32,sk=1,sw=0,dr=0,tm=1,oc=2"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --variant conv_umma --params "$P,$3" --flags 0,16 >> $OUT/ovh.log 2>&1
  timeout 120 python tools/run_op.py --row $1 --batch $2 --variant conv_umma --params "$P,$3" --reps 7 >> $OUT/cold.log 2>&1
done
cat $OUT/ovh.log; cat $OUT/cold.log
