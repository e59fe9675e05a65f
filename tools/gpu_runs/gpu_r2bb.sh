#!/bin/bash
# r2bb: fused 3xTF32 issue (2 MMAs per K step) for OCC-1 tiles with BN <= 96: parity, re-time all DB choices, first layers, bench
OUT=gpurun_out/r2bb; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bf16_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
timeout 900 python tools/db_retime.py --csv $OUT/retime_fp32.csv > $OUT/retime_fp32.log 2>&1; tail -1 $OUT/retime_fp32.log; grep -c FAIL $OUT/retime_fp32.log
timeout 600 python tools/try_params.py --ops 35:20,33:20,35:5 --params "BN=64,sk=1,sw=0,dr=0,tm=1" "BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" \
  "BN=96,sk=1,sw=0,dr=0,tm=6,cl=3" "BN=64,sk=1,sw=0,dr=0,tm=1,cl=3" "BN=96,sk=1,sw=0,dr=0,tm=6" > $OUT/try_first.log 2>&1; cat $OUT/try_first.log | cut -c1-110
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));c=d['config'];print('fp32',d['value'],d['ms_per_step'],c['per_batch_ms_back_to_back'])"
