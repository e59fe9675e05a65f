#!/bin/bash
# r2bm: e2e with input-heavy / output-heavy ops interleaved (bench default line, twice)
OUT=gpurun_out/r2bm; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
for i in 1 2; do
timeout 900 python bench.py --no-cpu > $OUT/bench_$i.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench_$i.json'));e=d['e2e'];print('fp32',d['value'],'e2e',e['value'],e['ms_per_step'],e['copy_bound_ms'],e['frac_of_copy_bound'])"
done
