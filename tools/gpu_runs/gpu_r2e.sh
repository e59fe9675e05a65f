# concurrent-step DB selection: latency-optimal vs SM-time-weighted tunes
OUT=gpurun_out/r2e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for DB in scratch/*.tsv; do
  n=$(basename $DB .tsv)
  for S in 4 8; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --streams $S --db $DB > $OUT/b_${n}_s$S.json 2> $OUT/b_${n}_s$S.err
    python -c "import json;d=json.load(open('$OUT/b_${n}_s$S.json'));print('$n s$S', d['value'],d['ms_per_step'],d['config']['serial_ms_per_step_rank0'])"
  done
done
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python tools/sanitize_ops.py > $OUT/sanitize_initcheck.log 2>&1; echo "exit $?" >> $OUT/sanitize_initcheck.log
tail -3 $OUT/sanitize_initcheck.log
