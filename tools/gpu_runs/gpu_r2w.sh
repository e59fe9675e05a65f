#!/bin/bash
# r2w: re-tune fp32 (now with conv_wino candidates) and tune the fp8 mode; re-pick sweep DBs; bench both
OUT=gpurun_out/r2w; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for P in 0 2; do
  n=$([ $P = 0 ] && echo fp32 || echo fp8)
  timeout 1500 python tools/tune_sweep.py --prec $P --out $OUT/tunedb_b200_$n.tsv --batches 1,2,3,5,10,20 --all-out $OUT/cands_$n.csv > $OUT/tune_$n.log 2>&1
  tail -1 $OUT/tune_$n.log
  python tools/pick_db.py --cands $OUT/cands_$n.csv --out $OUT/tunedb_b200_${n}_sweep.tsv --alpha 0.5 --slack 3
  cp $OUT/tunedb_b200_$n.tsv $OUT/tunedb_b200_${n}_sweep.tsv paper_1611_06945_b200/data/
  gzip -f $OUT/cands_$n.csv
done
grep -c conv_wino $OUT/tunedb_b200_fp32.tsv $OUT/tunedb_b200_fp32_sweep.tsv
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print('fp32',d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['roofline']['achieved'])"
timeout 600 python bench.py --steps 20 --warmup 5 --prec fp8 --no-cpu --no-e2e --per-op-out $OUT/per_op_fp8.csv > $OUT/bench_fp8.json 2> $OUT/bench_fp8.err
python -c "import json;d=json.load(open('$OUT/bench_fp8.json'));print('fp8',d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['roofline']['achieved'])"
timeout 600 python bench.py --steps 20 --warmup 5 --prec bf16 --no-cpu --no-e2e > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err
python -c "import json;d=json.load(open('$OUT/bench_bf16.json'));print('bf16',d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['roofline']['achieved'])"
