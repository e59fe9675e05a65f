#!/bin/bash
# r2ay: fc (MODE 1) weight boxes prefetched into L2 ahead of the shared-memory ring: distance sweep on fc6 / fc7
OUT=gpurun_out/r2ay; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
for A in 0 4 8 16 32; do
  echo "== B2C_L2_AHEAD=$A"
  B2C_L2_AHEAD=$A timeout 600 python tools/try_params.py --ops 25:20,25:5,13:20,13:5,25:10 --params \
    "conv_fc:BN=32,sk=8,sw=1,dr=0,tm=1,oc=2" "conv_fc:BN=32,sk=8,sw=1,dr=0,tm=1" "conv_fc:BN=32,sk=0,sw=1,dr=0,tm=1" \
    "conv_fc:BN=32,sk=4,sw=1,dr=0,tm=1,oc=2" "conv_fc:BN=64,sk=8,sw=1,dr=0,tm=1"
done > $OUT/fc_l2ahead.log 2>&1
grep -E "==|us" $OUT/fc_l2ahead.log | awk '{print $1, $2, $3, $4, $5}'
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "golden or fc" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
