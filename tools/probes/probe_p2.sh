OUT=gpurun_out/p2
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "34 20 BN=96,sk=1,sw=0" "35 20 BN=64,sk=1,sw=0" "33 1 BN=96,sk=1,sw=0"; do set -- $spec
  timeout 60 python tools/stress_op.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" --flush --iters 20 >> $OUT/stress.log 2>&1 || echo "exit $? $spec" >> $OUT/stress.log
done
for spec in "20 20 BN=96,sk=1,sw=0" "34 20 BN=96,sk=1,sw=0" "35 20 BN=64,sk=1,sw=0"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" --flags 0,16,18,22 >> $OUT/ovh.log 2>&1
done
for spec in "20 20 BN=96,sk=1,sw=0" "35 20 BN=64,sk=1,sw=0"; do set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" --flags 1 2>&1 | grep -v "rep0" >> $OUT/trace.log
done
