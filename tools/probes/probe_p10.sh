OUT=gpurun_out/p10
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "40 1 BN=32,sk=8,sw=1,dr=0,tm=1" "37 20 BN=96,sk=2,sw=1,dr=0,tm=1" "36 1 BN=32,sk=8,sw=1,dr=0,tm=1" "25 1 BN=32,sk=4,sw=1,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3" --flags 0 >> $OUT/ovh.log 2>&1
done
timeout 60 python tools/stress_op.py --row 37 --batch 20 --params "$P,BN=96,sk=2,sw=1,dr=0,tm=1" --flush --iters 10 >> $OUT/stress.log 2>&1
