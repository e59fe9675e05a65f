OUT=gpurun_out/r2g; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python tools/tune_sweep.py --prec 1 --out $OUT/tunedb_b200_bf16.tsv --batches 1,2,3,5,10,20 --all-out $OUT/cands_bf16.csv > $OUT/tune_bf16.log 2>&1
tail -1 $OUT/tune_bf16.log
python tools/pick_db.py --cands $OUT/cands_bf16.csv --out paper_1611_06945_b200/data/tunedb_b200_bf16_sweep.tsv --alpha 0.5 --slack 3
cp $OUT/tunedb_b200_bf16.tsv paper_1611_06945_b200/data/tunedb_b200_bf16.tsv
timeout 600 python bench.py --steps 20 --warmup 5 --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['ms_per_step'],d['config']['serial_ms_per_step_rank0'],d['e2e']['value'],d['cpu_baseline']['value'])"
timeout 600 python bench.py --steps 20 --warmup 5 --prec bf16 --no-cpu > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err
python -c "import json;d=json.load(open('$OUT/bench_bf16.json'));print('bf16',d['value'],d['ms_per_step'],d['config']['serial_ms_per_step_rank0'])"
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -8 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
