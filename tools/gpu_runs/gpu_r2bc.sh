#!/bin/bash
# r2bc: full fp32 re-tune with the fused-issue kernels (latency DB + re-picked sweep DB), bench old vs new DBs twice
OUT=gpurun_out/r2bc; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 2400 python tools/tune_sweep.py --prec 0 --out $OUT/tunedb_b200_fp32.tsv --batches 1,2,3,5,10,20 --all-out $OUT/cands_fp32.csv > $OUT/tune_fp32.log 2>&1
tail -1 $OUT/tune_fp32.log
python tools/pick_db.py --cands $OUT/cands_fp32.csv --out $OUT/tunedb_b200_fp32_sweep.tsv --alpha 0.5 --slack 3
gzip -f $OUT/cands_fp32.csv
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench_old_$i.json 2> /dev/null
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 --db $OUT/tunedb_b200_fp32.tsv --sweep-db $OUT/tunedb_b200_fp32_sweep.tsv > $OUT/bench_new_$i.json 2> /dev/null
python -c "import json;o=json.load(open('$OUT/bench_old_$i.json'));n=json.load(open('$OUT/bench_new_$i.json'));print('old',o['value'],o['ms_per_step'],o['config']['per_batch_ms_back_to_back'],'new',n['value'],n['ms_per_step'],n['config']['per_batch_ms_back_to_back'])"
done
