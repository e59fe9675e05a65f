OUT=gpurun_out/tma9
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "17 1 BN=32,sk=1,sw=0" "17 20 BN=128,sk=1,sw=0" "27 20 BN=128,sk=1,sw=0" "20 20 BN=96,sk=1,sw=0" "6 20 BN=64,sk=1,sw=0"; do set -- $spec
  for tm in 1 2; do
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=$tm" --flags 1 2>&1 | grep -v "rep0" >> $OUT/trace.log
  done
done
timeout 900 python -m pytest tests -q -m gpu -x -k golden > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
