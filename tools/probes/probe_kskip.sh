OUT=gpurun_out/ks1
mkdir -p $OUT
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log; grep -E "^(E |FAILED)" $OUT/pytest.log | head -5
B2C_NO_KSKIP=1 timeout 600 python bench.py --no-cpu --per-op-out $OUT/per_op_noskip.csv > $OUT/bench_noskip.json 2> $OUT/bench_noskip.err
timeout 600 python bench.py --no-cpu --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python - <<'PY'
import json
for f in ("gpurun_out/ks1/bench_noskip.json","gpurun_out/ks1/bench.json"):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d["value"], d["ms_per_step"], d["config"]["per_batch_ms"], d["e2e"]["value"], d["e2e"]["ms_per_step"])
PY
