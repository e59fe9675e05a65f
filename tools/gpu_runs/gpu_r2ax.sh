#!/bin/bash
# r2ax: step-level sweep-DB search with paired A/B timing (fp32, 4 alternatives per op), bench old vs new twice
OUT=gpurun_out/r2ax; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
D=paper_1611_06945_b200/data
timeout 3000 python tools/step_search.py --cands profiles/r2ar/cands_fp32_merged.csv.gz --db $D/tunedb_b200_fp32_sweep.tsv \
   --out $OUT/tunedb_b200_fp32_sweep.tsv --alts 4 --passes 1 --min-gain 0.003 > $OUT/search.log 2>&1; cat $OUT/search.log | tail -30
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench_old_$i.json 2> /dev/null
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 --sweep-db $OUT/tunedb_b200_fp32_sweep.tsv > $OUT/bench_new_$i.json 2> /dev/null
python -c "import json;o=json.load(open('$OUT/bench_old_$i.json'));n=json.load(open('$OUT/bench_new_$i.json'));print('old',o['value'],o['ms_per_step'],'new',n['value'],n['ms_per_step'])"
done
