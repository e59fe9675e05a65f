#!/bin/bash
# r2aq: sweep-DB pick parameters (alpha, slack) for the concurrent step, fp32 and bf16
OUT=gpurun_out/r2aq; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
for A in 0.25 0.5 0.75 1.0; do for SL in 2 3 5; do
  python tools/pick_db.py --cands profiles/r2al/cands_fp32.csv.gz --out $OUT/sw_fp32_${A}_${SL}.tsv --alpha $A --slack $SL > /dev/null
  timeout 300 python bench.py --sweep-db $OUT/sw_fp32_${A}_${SL}.tsv --no-cpu --no-e2e --steps 30 > $OUT/b_fp32_${A}_${SL}.json 2> /dev/null
  python -c "import json;d=json.load(open('$OUT/b_fp32_${A}_${SL}.json'));print('fp32 alpha $A slack $SL',d['value'],d['ms_per_step'])"
done; done
