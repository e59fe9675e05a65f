OUT=gpurun_out/tma8
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for pr in "BN=32,sk=4,sw=1" "BN=128,sk=4,sw=0" "BN=128,sk=1,sw=0"; do
    timeout 60 python tools/stress_op.py --row 25 --batch 20 --params "$P,$pr,dr=0,tm=1" --flush >> $OUT/stress.log 2>&1 || echo "exit $? $pr" >> $OUT/stress.log
done
timeout 60 python tools/stress_op.py --row 42 --batch 20 --params "$P,BN=128,sk=1,sw=0,dr=0,tm=1" --flush >> $OUT/stress.log 2>&1
timeout 60 python tools/stress_op.py --row 17 --batch 1 --params "$P,BN=32,sk=4,sw=0,dr=0,tm=1" --flush >> $OUT/stress.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
for spec in "17 1 BN=32,sk=1,sw=0" "42 20 BN=128,sk=1,sw=0"; do set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" --flags 1 2>&1 | grep -v "rep0" >> $OUT/trace.log
done
