set -x
OUT=gpurun_out/small
mkdir -p $OUT
for spec in "6 1" "0 1" "17 1"; do set -- $spec
  python tools/run_op.py --row $1 --batch $2 --reps 3 >> $OUT/times.log 2>&1
  ncu --set full --clock-control none --import-source on -k "regex:k_umma" -s 2 -c 1 -o $OUT/prof_r$1_n$2 python tools/run_op.py --row $1 --batch $2 --reps 3 > $OUT/ncu_r$1.log 2>&1
done
cat $OUT/times.log
