# small-op latency probe: cuDNN comparator, warm-L2 graph per-launch times, CTA-0 phase traces
OUT=gpurun_out/small1
mkdir -p $OUT
timeout 600 python tools/cudnn_compare.py --out $OUT/cudnn_per_op.csv > $OUT/cudnn.log 2>&1
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "6 1 conv_1x1 BN=32,sk=1,sw=0,dr=0" "0 1 conv_umma BN=32,sk=4,sw=0,dr=0,tm=1" "17 1 conv_1x1 BN=32,sk=1,sw=0,dr=0,tm=1" "38 1 conv_umma BN=32,sk=4,sw=0,dr=0,tm=1" "25 1 conv_umma BN=32,sk=4,sw=1,dr=0,tm=1" "13 1 conv_fc BN=32,sk=4,sw=1,dr=0,tm=2"; do set -- $spec
  timeout 120 python tools/op_overhead.py --row $1 --batch $2 --variant $3 --params "$P,$4" --flags 0 >> $OUT/ovh.log 2>&1
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --variant $3 --params "$P,$4" >> $OUT/trace.log 2>&1
done
