#!/bin/bash
# r2bu: shipped DBs with the BN=16 fc picks: signed 129-op sweep through both DBs, paired benches vs the previous DBs
OUT=gpurun_out/r2bu; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
true
cp scratch/old_lat.tsv $OUT/old_lat.tsv
cp scratch/old_sw.tsv $OUT/old_sw.tsv
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench_new_$i.json 2> /dev/null
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 --db $OUT/old_lat.tsv --sweep-db $OUT/old_sw.tsv > $OUT/bench_old_$i.json 2> /dev/null
python -c "import json;o=json.load(open('$OUT/bench_old_$i.json'));n=json.load(open('$OUT/bench_new_$i.json'));print('old',o['value'],o['config']['per_batch_ms_back_to_back'],'| new',n['value'],n['config']['per_batch_ms_back_to_back'])"
done
