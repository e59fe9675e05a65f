OUT=gpurun_out/as1
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 600 python bench.py --no-cpu --no-e2e --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err; cat $OUT/bench.json | head -c 900; echo
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "38 1 conv_umma BN=32,sk=4,sw=0,dr=0,tm=1" "42 20 conv_umma BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" "42 20 conv_umma BN=128,sk=1,sw=0,dr=0,tm=1" "25 1 conv_umma BN=32,sk=4,sw=1,dr=0,tm=1"; do set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --variant $3 --params "$P,$4" >> $OUT/trace.log 2>&1
done
grep "^time" $OUT/trace.log
