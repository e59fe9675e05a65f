OUT=gpurun_out/p6
mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "20 20 BN=96,sk=1,sw=0,dr=0,tm=1" "42 20 BN=128,sk=1,sw=0,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --params "$P,$3" --flags 1 2>&1 | grep -v "rep0" | grep "drain/epi\|time" >> $OUT/trace.log
done
for spec in "42 20 BN=128,sk=1,sw=0,dr=0,tm=1" "34 20 BN=96,sk=1,sw=0,dr=0,tm=1" "35 20 BN=64,sk=1,sw=0,dr=0,tm=1" "41 20 BN=192,sk=1,sw=0,dr=0,tm=1" "20 20 BN=96,sk=1,sw=0,dr=0,tm=1" "6 20 BN=64,sk=1,sw=0,dr=0,tm=1" "17 1 BN=32,sk=4,sw=0,dr=0,tm=1" "6 1 BN=32,sk=1,sw=0,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3" --flags 0 >> $OUT/ovh.log 2>&1
done
