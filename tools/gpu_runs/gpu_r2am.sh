#!/bin/bash
# r2am: fused 3xTF32 MMA issue (BN=32/64): re-time the shipped DB choices, e2e PCIe probe, GPU suite, bench
OUT=gpurun_out/r2am; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python tools/db_retime.py --csv $OUT/retime_fp32.csv > $OUT/retime_fp32.log 2>&1; tail -1 $OUT/retime_fp32.log
grep -c FAIL $OUT/retime_fp32.log
timeout 600 python tools/e2e_probe.py > $OUT/e2e_probe.log 2>&1; cat $OUT/e2e_probe.log | tail -14
timeout 1800 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 900 python bench.py --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print('fp32',d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['roofline']['achieved'],d['e2e']['value'],d['clocks'])"
P='MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,'
timeout 300 python tools/trace_op.py --row 0 --batch 1 --params "${P}BN=32,sk=4,sw=0,dr=0,tm=4" > $OUT/trace_row0.log 2>&1
timeout 300 python tools/trace_op.py --row 0 --batch 1 --params "${P}BN=32,sk=4,sw=0,dr=0,tm=4" --flags 3 >> $OUT/trace_row0.log 2>&1
timeout 300 python tools/trace_op.py --row 0 --batch 1 --params "${P}BN=32,sk=4,sw=0,dr=0,tm=4" --flags 9 >> $OUT/trace_row0.log 2>&1
timeout 300 python tools/trace_op.py --row 25 --batch 20 --variant conv_fc --params "${P}BN=32,sk=8,sw=1,dr=0,tm=1,oc=2" > $OUT/trace_fc6.log 2>&1
