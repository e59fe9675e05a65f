#!/bin/bash
# r2ar: k_fc_bulk (conv_fc_stream Kb=3): parity, timing vs the DB choices, re-tune fc6/fc7 rows, bench
OUT=gpurun_out/r2ar; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fc_bulk or fc_stream or golden" > $OUT/pytest_fc.log 2>&1; tail -2 $OUT/pytest_fc.log
timeout 600 python tools/try_params.py --ops 25:1,25:2,25:3,25:5,25:8,13:1,13:3,13:5,13:8 --params \
  "conv_fc_stream:MNt=1:1,MNb=8:1,Kb=3,vw=1" "conv_fc_stream:MNt=1:2,MNb=4:1,Kb=1,vw=1" "conv_fc_stream:MNt=1:4,MNb=4:1,Kb=1,vw=1" \
  "conv_fc:BN=32,sk=8,sw=1,dr=0,tm=1,oc=2" > $OUT/fc_try.log 2>&1; cat $OUT/fc_try.log
D=paper_1611_06945_b200/data
timeout 1200 python tools/tune_sweep.py --prec 0 --rows 13,25 --merge $D/tunedb_b200_fp32.tsv --out $OUT/tunedb_b200_fp32.tsv \
    --batches 1,2,3,5,10,20 --all-out $OUT/cands_new_fp32.csv > $OUT/tune_fp32.log 2>&1
cat $OUT/tune_fp32.log
python tools/merge_cands.py profiles/r2al/cands_fp32.csv.gz $OUT/cands_new_fp32.csv $OUT/cands_fp32.csv
python tools/pick_db.py --cands $OUT/cands_fp32.csv --out $OUT/tunedb_b200_fp32_sweep.tsv --alpha 0.5 --slack 3
cp $OUT/tunedb_b200_fp32.tsv $OUT/tunedb_b200_fp32_sweep.tsv $D/
gzip -f $OUT/cands_fp32.csv $OUT/cands_new_fp32.csv
timeout 900 python bench.py --per-op-out $OUT/per_op.csv --no-cpu > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));c=d['config'];print('fp32',d['value'],d['ms_per_step'],c['per_batch_ms_isolated'],c['per_batch_ms_back_to_back'],d['e2e']['value'])"
