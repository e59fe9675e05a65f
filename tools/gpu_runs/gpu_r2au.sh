#!/bin/bash
# r2au: SS path no longer commits the unused TMEM A-slot barrier (synccheck "missing wait"): synccheck over every family, bf16 parity, bf16 bench
OUT=gpurun_out/r2au; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_ops.py > $OUT/sanitize_synccheck.log 2>&1; echo "exit $?" >> $OUT/sanitize_synccheck.log
echo "synccheck: $(grep -E 'ERROR SUMMARY|sanitize_ops:' $OUT/sanitize_synccheck.log | tr '\n' ' ') $(tail -1 $OUT/sanitize_synccheck.log)"
timeout 900 python -m pytest tests/test_bf16_gpu.py -m gpu -x -q > $OUT/pytest_bf16.log 2>&1; tail -1 $OUT/pytest_bf16.log
timeout 600 python bench.py --prec bf16 --no-cpu --no-e2e > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err
python -c "import json;print('bf16',json.load(open('$OUT/bench_bf16.json'))['value'])"
