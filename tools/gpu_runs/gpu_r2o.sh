#!/bin/bash
# r2o: re-tune the fp32 DBs with the 2-SM pair candidates, re-pick the sweep DB, bench
OUT=gpurun_out/r2o; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python tools/tune_sweep.py --prec 0 --out $OUT/tunedb_b200_fp32.tsv --batches 1,2,3,5,10,20 --all-out $OUT/cands_fp32.csv > $OUT/tune_fp32.log 2>&1
tail -1 $OUT/tune_fp32.log
python tools/pick_db.py --cands $OUT/cands_fp32.csv --out $OUT/tunedb_b200_fp32_sweep.tsv --alpha 0.5 --slack 3
cp $OUT/tunedb_b200_fp32.tsv $OUT/tunedb_b200_fp32_sweep.tsv paper_1611_06945_b200/data/
gzip -kf $OUT/cands_fp32.csv
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['roofline']['achieved'],d['roofline']['kernel'])"
