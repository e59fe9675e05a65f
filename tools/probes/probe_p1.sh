OUT=gpurun_out/p1
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -25 $OUT/pytest_gpu.log
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "25 20 BN=32,sk=4,sw=1" "42 20 BN=128,sk=1,sw=0" "17 1 BN=32,sk=4,sw=0" "34 20 BN=96,sk=1,sw=0" "35 20 BN=64,sk=1,sw=0" "33 1 BN=96,sk=1,sw=0"; do set -- $spec
  timeout 60 python tools/stress_op.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" --flush --iters 20 >> $OUT/stress.log 2>&1 || echo "exit $? $spec" >> $OUT/stress.log
done
for spec in "42 20 BN=128,sk=1,sw=0" "20 20 BN=96,sk=1,sw=0" "6 20 BN=64,sk=1,sw=0" "34 20 BN=96,sk=1,sw=0" "35 20 BN=64,sk=1,sw=0" "33 5 BN=96,sk=1,sw=0" "17 1 BN=32,sk=4,sw=0" "40 20 BN=192,sk=2,sw=0" "41 20 BN=192,sk=1,sw=0"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" --flags 0 >> $OUT/ovh.log 2>&1
  timeout 120 python tools/run_op.py --row $1 --batch $2 --variant conv_umma --params "$P,$3,dr=0,tm=1" --reps 3 >> $OUT/times.log 2>&1
done
