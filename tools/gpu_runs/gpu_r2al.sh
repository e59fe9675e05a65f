#!/bin/bash
# r2al: re-tune fp32 (tm=6 candidates), full validation: pytest -m gpu, smoke, default bench, bf16/fp8 bench, reference arm
OUT=gpurun_out/r2al; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python tools/tune_sweep.py --prec 0 --out $OUT/tunedb_b200_fp32.tsv --batches 1,2,3,5,10,20 --all-out $OUT/cands_fp32.csv > $OUT/tune_fp32.log 2>&1
tail -1 $OUT/tune_fp32.log
python tools/pick_db.py --cands $OUT/cands_fp32.csv --out $OUT/tunedb_b200_fp32_sweep.tsv --alpha 0.5 --slack 3
cp $OUT/tunedb_b200_fp32.tsv $OUT/tunedb_b200_fp32_sweep.tsv paper_1611_06945_b200/data/
gzip -f $OUT/cands_fp32.csv
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log; tail -1 $OUT/smoke.log
timeout 900 python bench.py --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print('fp32',d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['roofline']['achieved'],d['roofline']['kernel'],d['e2e']['value'],d['cpu_baseline']['value'],d['clocks'])"
timeout 600 python bench.py --prec bf16 --no-cpu --no-e2e > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err
timeout 600 python bench.py --prec fp8 --no-cpu --no-e2e > $OUT/bench_fp8.json 2> $OUT/bench_fp8.err
python -c "import json;[print(n,json.load(open(f'$OUT/bench_{n}.json'))['value']) for n in ('bf16','fp8')]"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch.log 2>&1
python tools/ncu_summary.py --launches $OUT/launches.csv > $OUT/launches.md 2>&1; head -30 $OUT/launches.md
timeout 1200 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
python -c "import json;d=json.load(open('$OUT/bench_reference.json'));print('reference',d['value'],d['ms_per_step'])"
