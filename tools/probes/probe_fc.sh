OUT=gpurun_out/fc2
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log; grep -E "^E " $OUT/pytest.log | head -3
timeout 900 python tools/tune_sweep.py --rows 13,25 --merge paper_1611_06945_b200/data/tunedb_b200_fp32.tsv --out $OUT/tunedb_b200_fp32.tsv > $OUT/tune.log 2>&1; cut -c1-200 $OUT/tune.log
timeout 600 python bench.py --db $OUT/tunedb_b200_fp32.tsv --no-cpu > $OUT/bench.json 2> $OUT/bench.err; python -c "
import json;d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['config']['per_batch_ms'], d['e2e']['value'])"
