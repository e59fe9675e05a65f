#!/bin/bash
# r2h: state check of the restored tree + tcgen05 issue-rate probes (1-SM and 2-SM UMMA)
OUT=gpurun_out/r2h; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 120 ./tools/mma_probe > $OUT/mma_probe.log 2>&1; echo "probe exit $?" >> $OUT/mma_probe.log
cat $OUT/mma_probe.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
/usr/bin/time -f "%e s" timeout 900 python bench.py --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
tail -1 $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['value'],d['ms_per_step'],d['config']['per_batch_ms_isolated'],d['e2e']['value'],d['cpu_baseline']['value'])"
/usr/bin/time -f "%e s" timeout 900 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
tail -1 $OUT/bench_reference.err; head -c 600 $OUT/bench_reference.json
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
