#!/bin/bash
# r2by: ncu --set full per kernel family on the final tree (the tuned DB choices + the FFMA alternative for first layers)
OUT=gpurun_out/r2by; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
cap() {  # name row batch kernel-regex [variant params]
  local name=$1 row=$2 batch=$3 kre=$4; shift 4
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 -o $OUT/$name \
     python tools/run_op.py --row $row --batch $batch --reps 3 "$@" > $OUT/$name.log 2>&1
  echo "$name: $(tail -1 $OUT/$name.log)"
}
cap dom_r42n20 42 20 "k_tconv"
cap k1_r6n20 6 20 "k_tconv"
cap k1_r18n20 18 20 "k_tconv"
cap first_r34n20 34 20 "k_tconv"
cap relayout4_r34n20 34 20 "k_to_nhwc4_pad"
cap tiled_r34n20 34 20 "k_tiled" --variant conv_tiled --params "MNt=4:4,MNb=16:8,Kb=16,vw=4,lf=1,li=1"
cap fcs_r25n1 25 1 "k_fc_stream"
cap fc_r25n20 25 20 "k_tconv"
cap fc_r13n5 13 5 "k_tconv|k_fc"
cap fc16_r25n5 25 5 "k_tconv"
cap k3_r40n20 40 20 "k_tconv"
cap relayout_r38n5 38 5 "k_nchw_to_nhwc"
cap k5_r29n20 29 20 "k_tconv"
python tools/ncu_summary.py $(for f in $OUT/*.ncu-rep; do echo --rep $f; done) > $OUT/ncu_summary.md 2>&1
wc -l $OUT/ncu_summary.md
# keep the summary and the dominant kernel's report (gpurun copies back <= 64 MiB)
for name in dom_r42n20 first_r34n20 tiled_r34n20 k1_r6n20 fc_r25n20; do
  ncu -i $OUT/$name.ncu-rep --page details --csv > $OUT/$name.details.csv 2>/dev/null
done
ncu -i $OUT/dom_r42n20.ncu-rep --page raw --csv > $OUT/dom_r42n20.raw.csv 2>/dev/null
ls -la $OUT/*.ncu-rep
find $OUT -name "*.ncu-rep" ! -name "dom_r42n20.ncu-rep" -delete
du -sh $OUT
