OUT=gpurun_out/tune2
mkdir -p $OUT
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log; grep -E "^(E |FAILED)" $OUT/pytest.log | head -5
timeout 2400 python tools/tune_sweep.py --out $OUT/tunedb_b200_fp32.tsv > $OUT/tune.log 2>&1; tail -2 $OUT/tune.log
timeout 600 python bench.py --db $OUT/tunedb_b200_fp32.tsv --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err; head -c 700 $OUT/bench.json; echo
timeout 600 python tools/net_bench.py --db $OUT/tunedb_b200_fp32.tsv > $OUT/net_bench.jsonl 2>&1; cut -c1-120 $OUT/net_bench.jsonl
