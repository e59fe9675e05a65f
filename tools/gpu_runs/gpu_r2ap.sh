#!/bin/bash
# r2ap: concurrent-branch count of the sweep step; bench with back-to-back per-op times
OUT=gpurun_out/r2ap; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
for S in 8 12 16 24 32; do
  timeout 600 python bench.py --streams $S --no-cpu --no-e2e --steps 30 > $OUT/bench_s$S.json 2> $OUT/bench_s$S.err
  python -c "import json;d=json.load(open('$OUT/bench_s$S.json'));print('streams $S',d['value'],d['ms_per_step'])"
done
timeout 900 python bench.py --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));c=d['config'];print('fp32',d['value'],d['ms_per_step'],c['per_batch_ms_isolated'],c['per_batch_ms_back_to_back'],d['e2e']['value'],d['e2e']['frac_of_copy_bound'],d['clocks'])"
