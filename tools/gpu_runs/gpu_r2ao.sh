#!/bin/bash
# r2ao: first-layer space-to-depth (tm=6) in the bf16 / fp8 modes: parity, re-tune the first-layer rows, bench
OUT=gpurun_out/r2ao; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_bf16_gpu.py tests/test_fp8_gpu.py tests/test_gpu_parity.py -m gpu -x -q > $OUT/pytest_modes.log 2>&1; tail -2 $OUT/pytest_modes.log
D=paper_1611_06945_b200/data
for P in 1 2; do
  n=$([ $P = 1 ] && echo bf16 || echo fp8)
  old=$([ $P = 1 ] && echo profiles/r2ai/cands_bf16.csv.gz || echo profiles/r2aj/cands_fp8.csv.gz)
  timeout 1200 python tools/tune_sweep.py --prec $P --rows 33,34,35 --merge $D/tunedb_b200_$n.tsv --out $OUT/tunedb_b200_$n.tsv \
      --batches 1,2,3,5,10,20 --all-out $OUT/cands_new_$n.csv > $OUT/tune_$n.log 2>&1
  tail -1 $OUT/tune_$n.log
  python tools/merge_cands.py $old $OUT/cands_new_$n.csv $OUT/cands_$n.csv
  python tools/pick_db.py --cands $OUT/cands_$n.csv --out $OUT/tunedb_b200_${n}_sweep.tsv --alpha 0.5 --slack 3
  cp $OUT/tunedb_b200_$n.tsv $OUT/tunedb_b200_${n}_sweep.tsv $D/
  gzip -f $OUT/cands_$n.csv $OUT/cands_new_$n.csv
done
grep -E "k11|k7:s2" $D/tunedb_b200_bf16.tsv $D/tunedb_b200_fp8.tsv | head -30
timeout 600 python bench.py --prec bf16 --no-cpu --no-e2e --per-op-out $OUT/per_op_bf16.csv > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err
timeout 600 python bench.py --prec fp8 --no-cpu --no-e2e --per-op-out $OUT/per_op_fp8.csv > $OUT/bench_fp8.json 2> $OUT/bench_fp8.err
python -c "import json;[print(n,json.load(open(f'$OUT/bench_{n}.json'))['value'],json.load(open(f'$OUT/bench_{n}.json'))['roofline']['op']) for n in ('bf16','fp8')]"
