#!/bin/bash
OUT=gpurun_out/r2r; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:wino|k_tconv" -s 3 -c 3 -o $OUT/wino40 \
  python tools/try_params.py --ops 40:20 --params conv_wino:BN=128,sk=1,sw=1,tm=1 --reps 2 > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py --rep $OUT/wino40.ncu-rep > $OUT/wino40.md 2>&1
cat $OUT/wino40.md
for k in k_wino_input k_wino_output; do
ncu -i $OUT/wino40.ncu-rep --page details -k $k --csv 2>/dev/null | grep -i "stall\|Throughput\|Warp Cycles\|Achieved Occ\|Eligible\|Issued" | head -30 > $OUT/$k.details.csv
cat $OUT/$k.details.csv | cut -c1-220
done
