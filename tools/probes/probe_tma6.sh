OUT=gpurun_out/tma6
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "17 1 BN=32,sk=1,sw=0" "42 20 BN=128,sk=1,sw=0"; do set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" --flags 1 2>&1 | grep -v "rep0" >> $OUT/trace.log
done
for spec in "42 20 BN=128,sk=1,sw=0" "6 1 BN=32,sk=1,sw=0" "0 1 BN=32,sk=1,sw=0" "17 1 BN=32,sk=1,sw=0" "17 1 BN=32,sk=4,sw=0" "25 20 BN=32,sk=4,sw=1" "13 20 BN=32,sk=4,sw=1" "40 20 BN=96,sk=1,sw=0" "41 20 BN=192,sk=1,sw=0"; do set -- $spec
  for tm in 0 1; do
  timeout 120 python tools/run_op.py --row $1 --batch $2 --variant conv_umma --params "$P,$3,dr=0,tm=$tm" --reps 3 >> $OUT/times.log 2>&1
  done
done
timeout 120 python tools/run_op.py --row 25 --batch 20 --variant conv_fc --params "$P,BN=32,sk=4,sw=1,dr=0,tm=1" --reps 3 >> $OUT/times.log 2>&1
timeout 120 python tools/run_op.py --row 13 --batch 20 --variant conv_fc --params "$P,BN=32,sk=4,sw=1,dr=0,tm=1" --reps 3 >> $OUT/times.log 2>&1
