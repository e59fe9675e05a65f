# bottleneck experiments: per-op graph time with debug flags
#   2: hi*hi only (1/3 of the MMAs)  4: no B split  8: no A->TMEM  16: reuse the NHWC copy (no re-layout launch)
OUT=gpurun_out/r2c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
run() { timeout 120 python tools/op_overhead.py --row $1 --batch $2 --variant $3 --params "$P,$4" --flags 0,2,8,10,16,24,26 --k 30 >> $OUT/ovh.log 2>&1; }
run 42 20 conv_umma BN=128,sk=0,sw=0,dr=0,tm=1
run 42 20 conv_umma BN=192,sk=0,sw=0,dr=0,tm=1
run 42 20 conv_umma BN=128,sk=1,sw=0,dr=0,tm=1
run 40 20 conv_umma BN=128,sk=0,sw=0,dr=0,tm=1
run 41 20 conv_umma BN=192,sk=1,sw=0,dr=0,tm=4
run 4 20 conv_1x1 BN=128,sk=1,sw=0,dr=0,tm=3
run 4 20 conv_1x1 BN=64,sk=2,sw=0,dr=0,tm=3
run 38 1 conv_umma BN=32,sk=4,sw=0,dr=0,tm=1
run 17 1 conv_1x1 BN=32,sk=1,sw=0,dr=0,tm=1
run 34 20 conv_umma BN=96,sk=1,sw=0,dr=0,tm=1
cat $OUT/ovh.log
