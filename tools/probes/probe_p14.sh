OUT=gpurun_out/p14
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log; grep -E "^E " $OUT/pytest_gpu.log | head -3
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "42 20 BN=128,sk=1,sw=0,dr=0,tm=1" "34 20 BN=96,sk=1,sw=0,dr=0,tm=1" "17 1 BN=32,sk=4,sw=0,dr=0,tm=1" "20 20 BN=96,sk=1,sw=0,dr=0,tm=2"; do set -- $spec
  timeout 60 python tools/stress_op.py --row $1 --batch $2 --params "$P,$3" --flush --iters 20 >> $OUT/stress.log 2>&1 || echo "exit $? $spec" >> $OUT/stress.log
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3" --flags 0 >> $OUT/ovh.log 2>&1
  B2C_SEPARATE_NHWC=1 timeout 120 python tools/op_overhead.py --row $1 --batch $2 --params "$P,$3" --flags 0 | sed 's/^/SEP /' >> $OUT/ovh.log 2>&1
done
timeout 900 python bench.py --no-cpu --no-e2e > $OUT/bench.json 2>&1
python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'], d['ms_per_step'], d['config']['per_batch_ms'], d['gpu_launches'])"
