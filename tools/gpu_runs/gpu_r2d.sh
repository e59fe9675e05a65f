# sanitizers over every kernel family + full re-tune (batches incl. the shard-mode slab sizes) with all candidates
OUT=gpurun_out/r2d; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/sanitize_ops.py > $OUT/sanitize_plain.log 2>&1; echo "exit $?" >> $OUT/sanitize_plain.log
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_ops.py > $OUT/sanitize_$T.log 2>&1; echo "exit $?" >> $OUT/sanitize_$T.log
  tail -3 $OUT/sanitize_$T.log
done
timeout 1800 python tools/tune_sweep.py --out $OUT/tunedb_b200_fp32.tsv --batches 1,2,3,5,10,20 --all-out $OUT/cands_fp32.csv > $OUT/tune_fp32.log 2>&1
tail -2 $OUT/tune_fp32.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --db $OUT/tunedb_b200_fp32.tsv --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['ms_per_step'],d['config']['group_ms'],d['config']['serial_ms_per_step_rank0'])"
