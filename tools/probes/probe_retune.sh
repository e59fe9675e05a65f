OUT=gpurun_out/m8
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_host.py -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log; grep -E "^E " $OUT/pytest.log | head -6
timeout 2400 python tools/tune_sweep.py --out $OUT/tunedb_b200_fp32.tsv > $OUT/tune.log 2>&1; tail -1 $OUT/tune.log
timeout 2400 python tools/tune_sweep.py --prec 1 --out $OUT/tunedb_b200_bf16.tsv > $OUT/tune_bf16.log 2>&1; tail -1 $OUT/tune_bf16.log
timeout 600 python bench.py --db $OUT/tunedb_b200_fp32.tsv --no-cpu --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err; head -c 300 $OUT/bench.json; echo
timeout 600 python bench.py --prec bf16 --db $OUT/tunedb_b200_bf16.tsv --no-cpu --no-e2e > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err; head -c 300 $OUT/bench_bf16.json; echo
grep -c "tm=3" $OUT/tunedb_b200_fp32.tsv
