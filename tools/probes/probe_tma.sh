set -x
OUT=gpurun_out/tma1
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests -x -q -m gpu -k "golden and (case0 or case1 or case5 or case10 or case40 or case60 or case80)" > $OUT/golden_few.log 2>&1; tail -5 $OUT/golden_few.log
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -15 $OUT/pytest_gpu.log
for spec in "42 20 BN=128,sk=1,sw=0" "6 1 BN=32,sk=1,sw=0" "0 1 BN=32,sk=1,sw=0" "17 1 BN=32,sk=1,sw=0" "25 20 BN=32,sk=4,sw=1" "13 20 BN=32,sk=4,sw=1" "40 20 BN=96,sk=1,sw=0" "41 20 BN=192,sk=1,sw=0"; do set -- $spec
  for tm in 0 1; do
  timeout 120 python tools/run_op.py --row $1 --batch $2 --variant conv_umma --params "MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,$3,dr=0,tm=$tm" --reps 3 >> $OUT/times.log 2>&1
  done
done
cat $OUT/times.log
