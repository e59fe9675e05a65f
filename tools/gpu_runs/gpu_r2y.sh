#!/bin/bash
# r2y: full validation of the tree: pytest -m gpu, smoke, default bench (as the driver runs it), reference arm
OUT=gpurun_out/r2y; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log; tail -3 $OUT/smoke.log
S=$(date +%s); timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $? in $(( $(date +%s) - S )) s"
python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['cpu_baseline']['value'],d['clocks'])"
S=$(date +%s); timeout 1200 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "reference exit $? in $(( $(date +%s) - S )) s"
head -c 700 $OUT/bench_reference.json
