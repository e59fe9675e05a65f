OUT=gpurun_out/tune2
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 2400 python tools/tune_sweep.py --out $OUT/tunedb_b200_fp32.tsv > $OUT/tune.log 2>&1
tail -2 $OUT/tune.log
timeout 900 python bench.py --db $OUT/tunedb_b200_fp32.tsv --per-op-out $OUT/per_op.csv --no-cpu > $OUT/bench.json 2> $OUT/bench.err
cat $OUT/bench.json
