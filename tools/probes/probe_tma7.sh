OUT=gpurun_out/tma7
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for pr in "BN=32,sk=4,sw=1" "BN=32,sk=1,sw=1" "BN=128,sk=4,sw=0" "BN=64,sk=2,sw=1"; do
  for fl in "" "--flush"; do
    timeout 60 python tools/stress_op.py --row 25 --batch 20 --params "$P,$pr,dr=0,tm=1" $fl >> $OUT/stress.log 2>&1 || echo "exit $? $pr $fl" >> $OUT/stress.log
  done
done
timeout 60 python tools/stress_op.py --row 25 --batch 5 --params "$P,BN=32,sk=4,sw=1,dr=0,tm=1" --flush >> $OUT/stress.log 2>&1
timeout 60 python tools/stress_op.py --row 36 --batch 20 --params "$P,BN=96,sk=2,sw=0,dr=0,tm=1" --flush >> $OUT/stress.log 2>&1
timeout 60 python tools/stress_op.py --row 37 --batch 20 --params "$P,BN=96,sk=2,sw=1,dr=0,tm=1" --flush >> $OUT/stress.log 2>&1
