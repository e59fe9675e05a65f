OUT=gpurun_out/p3
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log; grep -E "Error|assert " $OUT/pytest_gpu.log | head -5
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "34 20 BN=96,sk=1,sw=0,dr=0,tm=1" "35 20 BN=64,sk=1,sw=0,dr=0,tm=1" "33 1 BN=96,sk=1,sw=0,dr=0,tm=1" "35 20 BN=64,sk=1,sw=0,dr=0,tm=2"; do set -- $spec
  timeout 60 python tools/stress_op.py --row $1 --batch $2 --params "$P,$3" --flush --iters 20 >> $OUT/stress.log 2>&1 || echo "exit $? $spec" >> $OUT/stress.log
done
for spec in "34 20 BN=96,sk=1,sw=0,dr=0,tm=1" "35 20 BN=64,sk=1,sw=0,dr=0,tm=1" "35 20 BN=64,sk=1,sw=0,dr=0,tm=2" "34 5 BN=96,sk=1,sw=0,dr=0,tm=1" "34 1 BN=96,sk=1,sw=0,dr=0,tm=1" "34 1 BN=32,sk=2,sw=0,dr=0,tm=1" "35 1 BN=64,sk=1,sw=0,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3" --flags 0,16 >> $OUT/ovh.log 2>&1
done
