OUT=gpurun_out/p22
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_tconv" -s 2 -c 1 -o $OUT/prof_r42 python tools/run_op.py --row 42 --batch 20 --variant conv_umma --params "$P,BN=128,sk=1,sw=0,dr=0,tm=1" --reps 3 > $OUT/ncu42.log 2>&1
