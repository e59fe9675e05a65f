#!/bin/bash
# r2bx: LPT branch dealing by SM-time instead of time (B2C_LPT_SMTIME): paired benches
OUT=gpurun_out/r2bx; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench_time_$i.json 2> $OUT/err
B2C_LPT_SMTIME=1 timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > $OUT/bench_smtime_$i.json 2>> $OUT/err
python -c "import json;o=json.load(open('$OUT/bench_time_$i.json'));n=json.load(open('$OUT/bench_smtime_$i.json'));print('LPT by time',o['value'],'| by SM-time',n['value'])"
done
