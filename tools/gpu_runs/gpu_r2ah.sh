#!/bin/bash
# r2ai: re-tune the bf16 DBs with the SS (tm=5) and SS-pair candidates; bench bf16 and fp32
OUT=gpurun_out/r2ai; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k golden > $OUT/pytest_golden.log 2>&1; tail -1 $OUT/pytest_golden.log
timeout 1500 python tools/tune_sweep.py --prec 1 --out $OUT/tunedb_b200_bf16.tsv --batches 1,2,3,5,10,20 --all-out $OUT/cands_bf16.csv > $OUT/tune_bf16.log 2>&1
tail -1 $OUT/tune_bf16.log
python tools/pick_db.py --cands $OUT/cands_bf16.csv --out $OUT/tunedb_b200_bf16_sweep.tsv --alpha 0.5 --slack 3
cp $OUT/tunedb_b200_bf16.tsv $OUT/tunedb_b200_bf16_sweep.tsv paper_1611_06945_b200/data/
gzip -f $OUT/cands_bf16.csv
grep -c "tm=5" $OUT/tunedb_b200_bf16.tsv $OUT/tunedb_b200_bf16_sweep.tsv
timeout 600 python bench.py --warmup 5 --prec bf16 --no-cpu --no-e2e --per-op-out $OUT/per_op_bf16.csv > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err
python -c "import json;d=json.load(open('$OUT/bench_bf16.json'));print('bf16',d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['roofline']['achieved'],d['roofline']['kernel'])"
timeout 600 python bench.py --warmup 5 --no-cpu --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print('fp32',d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['roofline']['achieved'],d['clocks'])"
