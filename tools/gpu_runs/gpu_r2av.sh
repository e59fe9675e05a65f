#!/bin/bash
# r2av: four drain warpgroups (DG = 4) for single-CTA BN >= 128 tiles: parity, re-time the DB choices, bench
OUT=gpurun_out/r2av; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bf16_gpu.py -m gpu -x -q > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
timeout 900 python tools/db_retime.py --csv $OUT/retime_fp32.csv > $OUT/retime_fp32.log 2>&1; tail -1 $OUT/retime_fp32.log
grep -c FAIL $OUT/retime_fp32.log
timeout 600 python bench.py --no-cpu --no-e2e --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));c=d['config'];print('fp32',d['value'],d['ms_per_step'],c['per_batch_ms_isolated'],c['per_batch_ms_back_to_back'])"
