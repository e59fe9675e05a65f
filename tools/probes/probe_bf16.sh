OUT=gpurun_out/bf1
mkdir -p $OUT
timeout 900 python -m pytest tests/test_bf16_gpu.py -x -q -m gpu > $OUT/pytest_bf16.log 2>&1; tail -3 $OUT/pytest_bf16.log; grep -E "^E " $OUT/pytest_bf16.log | head -8
