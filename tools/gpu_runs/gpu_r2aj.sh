#!/bin/bash
# r2aj: re-tune fp32 and fp8 (two loader warps, BN=96 pairs), re-pick, bench fp32 / fp8
OUT=gpurun_out/r2aj; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for P in 0 2; do
  n=$([ $P = 0 ] && echo fp32 || echo fp8)
  timeout 1500 python tools/tune_sweep.py --prec $P --out $OUT/tunedb_b200_$n.tsv --batches 1,2,3,5,10,20 --all-out $OUT/cands_$n.csv > $OUT/tune_$n.log 2>&1
  tail -1 $OUT/tune_$n.log
  python tools/pick_db.py --cands $OUT/cands_$n.csv --out $OUT/tunedb_b200_${n}_sweep.tsv --alpha 0.5 --slack 3
  cp $OUT/tunedb_b200_$n.tsv $OUT/tunedb_b200_${n}_sweep.tsv paper_1611_06945_b200/data/
  gzip -f $OUT/cands_$n.csv
done
timeout 600 python bench.py --warmup 5 --no-cpu --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print('fp32',d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['roofline']['achieved'],d['roofline']['kernel'],d['clocks'])"
timeout 600 python bench.py --warmup 5 --prec fp8 --no-cpu --no-e2e > $OUT/bench_fp8.json 2> $OUT/bench_fp8.err
python -c "import json;d=json.load(open('$OUT/bench_fp8.json'));print('fp8',d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'])"
