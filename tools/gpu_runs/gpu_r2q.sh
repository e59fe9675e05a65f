#!/bin/bash
OUT=gpurun_out/r2q; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/wino_launches.csv \
  python tools/try_params.py --ops 40:20,38:5 --params conv_wino:BN=128,sk=1,sw=1,tm=1 conv_wino:BN=128,sk=1,tm=1 --reps 2 > $OUT/ncu_try.log 2>&1
python tools/ncu_summary.py $OUT/wino_launches.csv 2>/dev/null | head -30 || true
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r2q/wino_launches.csv')))
hdr=None
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if 'wino' in d['Kernel Name'] or 'k_tconv' in d['Kernel Name']:
            print(d['ID'], d['Kernel Name'][:60], d['Metric Name'], d['Metric Value'])
PY
