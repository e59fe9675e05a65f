#!/bin/bash
# r2az: MODE 9 first-layer input patches (tm=7): parity, timings vs the shipped first-layer choices (fp32 / bf16 / fp8)
OUT=gpurun_out/r2az; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 300 python tools/sanitize_ops.py --only MODE9 > $OUT/san.log 2>&1; tail -2 $OUT/san.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "golden or space_to_depth" > $OUT/pytest_fp32.log 2>&1; tail -3 $OUT/pytest_fp32.log
timeout 900 python -m pytest tests/test_bf16_gpu.py tests/test_fp8_gpu.py -m gpu -x -q > $OUT/pytest_modes.log 2>&1; tail -3 $OUT/pytest_modes.log
timeout 900 python tools/try_params.py --ops 35:20,35:5,35:1,33:20,34:20,33:5,33:1 --params \
  "BN=64,sk=1,sw=0,dr=0,tm=1,oc=2" "BN=96,sk=1,sw=0,dr=0,tm=6,cl=3" \
  "BN=64,sk=1,sw=0,dr=0,tm=7" "BN=96,sk=1,sw=0,dr=0,tm=7" "BN=64,sk=0,sw=0,dr=0,tm=7" "BN=64,sk=1,sw=0,dr=0,tm=7,cl=3" \
  "BN=96,sk=1,sw=0,dr=0,tm=7,cl=3" "BN=32,sk=2,sw=0,dr=0,tm=7" "BN=128,sk=1,sw=0,dr=0,tm=7" > $OUT/try_fp32.log 2>&1; cat $OUT/try_fp32.log | cut -c1-120
timeout 900 python tools/try_params.py --ops 35:20,35:5,33:20,33:5 --params \
  "BN=64,sk=1,sw=0,dr=0,tm=1,pr=1" "BN=128,sk=1,sw=0,dr=0,tm=6,pr=1" "BN=64,sk=1,sw=0,dr=0,tm=7,pr=1" "BN=128,sk=1,sw=0,dr=0,tm=7,pr=1" \
  "BN=64,sk=0,sw=0,dr=0,tm=7,pr=1" "BN=64,sk=1,sw=0,dr=0,tm=7,pr=2" "BN=128,sk=1,sw=0,dr=0,tm=7,pr=2" "BN=64,sk=1,sw=0,dr=0,tm=1,pr=2" > $OUT/try_modes.log 2>&1; cat $OUT/try_modes.log | cut -c1-120
P='MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,'
timeout 120 python tools/trace_op.py --row 35 --batch 20 --params "${P}BN=64,sk=1,sw=0,dr=0,tm=7" > $OUT/trace_r35_tm7.log 2>&1
