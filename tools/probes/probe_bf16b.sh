OUT=gpurun_out/bf2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_bf16_gpu.py -x -q -m gpu -k full_size > $OUT/pytest_bf16.log 2>&1; tail -2 $OUT/pytest_bf16.log; grep -E "^E " $OUT/pytest_bf16.log | head -5
timeout 2400 python tools/tune_sweep.py --prec 1 --out $OUT/tunedb_b200_bf16.tsv > $OUT/tune.log 2>&1; tail -2 $OUT/tune.log
timeout 600 python bench.py --prec bf16 --db $OUT/tunedb_b200_bf16.tsv --no-cpu --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err; head -c 600 $OUT/bench.json; echo; tail -3 $OUT/bench.err
