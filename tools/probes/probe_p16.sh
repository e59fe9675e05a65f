OUT=gpurun_out/p16
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_tconv" -s 2 -c 1 -o $OUT/prof_r20 python tools/run_op.py --row 20 --batch 20 --variant conv_umma --params "$P,BN=96,sk=1,sw=0,dr=0,tm=2" --reps 3 > $OUT/ncu20.log 2>&1
timeout 120 python tools/trace_op.py --row 20 --batch 20 --params "$P,BN=96,sk=1,sw=0,dr=0,tm=2" --flags 1 2>&1 | grep -v "rep0" >> $OUT/trace.log
