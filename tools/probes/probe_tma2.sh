set -x
OUT=gpurun_out/tma2
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for spec in "6 1 BN=32,sk=1,sw=0" "0 1 BN=32,sk=1,sw=0" "17 1 BN=32,sk=1,sw=0" "42 20 BN=128,sk=1,sw=0" "13 20 BN=32,sk=4,sw=1"; do set -- $spec
  timeout 120 python tools/trace_op.py --row $1 --batch $2 --params "$P,$3,dr=0,tm=1" >> $OUT/trace.log 2>&1
done
cat $OUT/trace.log
timeout 300 compute-sanitizer --tool memcheck python tools/run_op.py --row 25 --batch 20 --variant conv_umma --params "$P,BN=32,sk=4,sw=1,dr=0,tm=1" --reps 1 > $OUT/sanitizer25.log 2>&1
tail -40 $OUT/sanitizer25.log
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; tail -15 $OUT/pytest_gpu.log
