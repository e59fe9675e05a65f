#!/bin/bash
# r2bw: ring depth cap 8 -> 12 (BN=16/32 single-CTA tiles get 9-11 stages): parity, re-time, bench
OUT=gpurun_out/r2bw; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
P='MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,'
for spec in "3 conv_1x1 BN=32,sk=4,sw=0,dr=0,tm=3" "0 conv_umma BN=32,sk=4,sw=0,dr=0,tm=4"; do
  set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch 1 --variant $2 --params "${P}$3" 2>&1 | head -4 | cut -c1-300
done > $OUT/traces.log; cat $OUT/traces.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fp8_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
timeout 900 python tools/db_retime.py --csv $OUT/retime_fp32.csv > $OUT/retime_fp32.log 2>&1; tail -1 $OUT/retime_fp32.log; grep -c FAIL $OUT/retime_fp32.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench_$i.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench_$i.json'));c=d['config'];print('fp32',d['value'],d['ms_per_step'],c['per_batch_ms_isolated'],c['per_batch_ms_back_to_back'])"
done
