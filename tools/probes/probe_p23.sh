OUT=gpurun_out/p23
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log; grep -E "^E " $OUT/pytest_gpu.log | head -3
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "42 20 BN=128,sw=0,dr=0,tm=1" "34 20 BN=96,sw=0,dr=0,tm=1" "35 20 BN=64,sw=0,dr=0,tm=1" "40 20 BN=96,sw=0,dr=0,tm=1" "41 20 BN=192,sw=0,dr=0,tm=1" "20 20 BN=96,sw=0,dr=0,tm=2" "40 5 BN=96,sw=0,dr=0,tm=1" "17 1 BN=32,sw=0,dr=0,tm=1" "40 1 BN=32,sw=1,dr=0,tm=1"; do set -- $spec
  for sk in 1 0; do
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3,sk=$sk" --flags 0 >> $OUT/ovh.log 2>&1
  done
  timeout 60 python tools/stress_op.py --row $1 --batch $2 --params "$P,$3,sk=0" --flush --iters 10 >> $OUT/stress.log 2>&1 || echo "exit $? $spec" >> $OUT/stress.log
done
