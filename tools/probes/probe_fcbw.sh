OUT=gpurun_out/fcbw
mkdir -p $OUT
P="MNt=1:4,MNb=4:1,Kb=1,vw=1,lf=1,li=1"
for spec in "13 1 conv_fc_stream MNt=1:4,MNb=4:1,Kb=1,vw=1" "13 1 conv_fc_stream MNt=1:8,MNb=2:1,Kb=1,vw=1" "13 1 conv_fc_stream MNt=1:2,MNb=8:1,Kb=2,vw=1" "25 1 conv_fc_stream MNt=1:2,MNb=4:1,Kb=1,vw=1" "25 5 conv_fc_stream MNt=1:2,MNb=8:1,Kb=2,vw=1" "25 20 conv_fc_stream MNt=1:2,MNb=8:1,Kb=2,vw=1" "25 20 conv_fc MNt=4:4,MNb=16:16,Kb=4,vw=4,BN=32,sk=8,sw=1,dr=0,tm=1,oc=2"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --variant $3 --params "$4" --flags 0 --k 20 >> $OUT/ovh.log 2>&1
  timeout 120 python tools/run_op.py --row $1 --batch $2 --variant $3 --params "$4" --reps 7 >> $OUT/cold.log 2>&1
done
cat $OUT/ovh.log $OUT/cold.log
