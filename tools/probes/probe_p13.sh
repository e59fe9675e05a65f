OUT=gpurun_out/p13
mkdir -p $OUT
timeout 900 python bench.py --no-cpu --no-e2e > $OUT/bench0.json 2>&1
timeout 900 python bench.py --no-cpu --no-e2e --debug-flags 16 --per-op-out $OUT/per_op16.csv > $OUT/bench16.json 2>&1
B2C_NO_PDL=1 timeout 900 python bench.py --no-cpu --no-e2e > $OUT/bench_nopdl.json 2>&1
for f in bench0 bench16 bench_nopdl; do python -c "import json;d=json.load(open('$OUT/$f.json'));print('$f', d['value'], d['ms_per_step'], d['config']['per_batch_ms'])"; done
