#!/bin/bash
# r2br: resident filter tiles (one filter tile with <= STAGES K blocks: loaded once per CTA, the ring carries pixel tiles only): parity, re-time, first layers, bench with / without
OUT=gpurun_out/r2br; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_bf16_gpu.py tests/test_fp8_gpu.py tests/test_gpu_signed_sweep.py tests/test_gpu_all_candidates.py -m gpu -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 300 python tools/sanitize_ops.py > $OUT/san.log 2>&1; tail -1 $OUT/san.log
timeout 900 python tools/db_retime.py --csv $OUT/retime_fp32.csv > $OUT/retime_fp32.log 2>&1; tail -1 $OUT/retime_fp32.log; grep -c FAIL $OUT/retime_fp32.log
timeout 600 python tools/try_params.py --ops 35:20,35:5,6:20,20:20,33:20 --params "BN=64,sk=1,sw=0,dr=0,tm=1" "BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" "BN=64,sk=1,sw=0,dr=0,tm=3" "BN=96,sk=1,sw=0,dr=0,tm=3" "BN=96,sk=1,sw=0,dr=0,tm=6,cl=3" > $OUT/try.log 2>&1; cat $OUT/try.log | cut -c1-110
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench_$i.json 2> $OUT/bench.err
B2C_NO_RESIDENT_B=1 timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench_norb_$i.json 2> /dev/null
python -c "import json;d=json.load(open('$OUT/bench_$i.json'));n=json.load(open('$OUT/bench_norb_$i.json'));c=d['config'];print('rb',d['value'],d['ms_per_step'],c['per_batch_ms_back_to_back'],'| no rb',n['value'],n['ms_per_step'],n['config']['per_batch_ms_back_to_back'])"
done
