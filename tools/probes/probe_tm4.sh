OUT=gpurun_out/tm4b
mkdir -p $OUT
P="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
for cs in twin00 twin29 twin31 twin39 twin41; do
  CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/probe_one.py --case $cs --params "$P,BN=32,sk=1,sw=0,dr=0,tm=4" >> $OUT/one.log 2>&1 || { echo "FAIL $cs"; tail -2 $OUT/one.log; exit 1; }
done
grep -E "ok|MISMATCH" $OUT/one.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bf16_gpu.py -x -q -m gpu > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log; grep -E "^E " $OUT/pytest.log | head -5
