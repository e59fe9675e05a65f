OUT=gpurun_out/pad
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bf16_gpu.py -x -q -m gpu > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log; grep -E "^E " $OUT/pytest.log | head -3
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "34 20 BN=96,sk=1,sw=0,dr=0,tm=1" "35 20 BN=64,sk=1,sw=0,dr=0,tm=1,oc=2"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --variant conv_umma --params "$P,$3" --flags 0,16 >> $OUT/ovh.log 2>&1
done
cat $OUT/ovh.log
timeout 600 python bench.py --no-cpu > $OUT/bench.json 2> $OUT/bench.err; python -c "
import json;d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['config']['per_batch_ms'], d['e2e']['value'])"
