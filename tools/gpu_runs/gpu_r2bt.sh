#!/bin/bash
# r2bt: 16-image swapped fc tile (BN=16): parity, fc timings, re-tune the fc rows, bench
OUT=gpurun_out/r2bt; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 600 python tools/try_params.py --ops 25:5,13:5,25:10,25:3,13:3,25:2 --params \
  "conv_fc:BN=32,sk=8,sw=1,dr=0,tm=1,oc=2" "conv_fc:BN=16,sk=8,sw=1,dr=0,tm=1,oc=2" "conv_fc:BN=16,sk=8,sw=1,dr=0,tm=1" \
  "conv_fc:BN=16,sk=4,sw=1,dr=0,tm=1,oc=2" "conv_fc:BN=16,sk=0,sw=1,dr=0,tm=1" "conv_fc:BN=16,sk=16,sw=1,dr=0,tm=1,oc=2" > $OUT/fc_try.log 2>&1; cat $OUT/fc_try.log | cut -c1-100
D=paper_1611_06945_b200/data
timeout 1200 python tools/tune_sweep.py --prec 0 --rows 13,25 --merge $D/tunedb_b200_fp32.tsv --out $OUT/tunedb_b200_fp32.tsv \
    --batches 1,2,3,5,10,20 --all-out $OUT/cands_new_fp32.csv > $OUT/tune_fp32.log 2>&1
grep -E "oc4096" $OUT/tune_fp32.log | cut -c1-170
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 --db $OUT/tunedb_b200_fp32.tsv > $OUT/bench_new.json 2> /dev/null
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench_old.json 2> /dev/null
python -c "import json;o=json.load(open('$OUT/bench_old.json'));n=json.load(open('$OUT/bench_new.json'));print('old',o['value'],o['config']['per_batch_ms_back_to_back'],'new latency DB',n['value'],n['config']['per_batch_ms_back_to_back'])"
