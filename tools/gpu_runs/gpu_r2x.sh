#!/bin/bash
# r2x: cluster split-K (DSMEM fixup) parity + small-op timings vs the L2-ticket fixup
OUT=gpurun_out/r2x; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or split_k or slabs" > $OUT/pytest_golden.log 2>&1; echo "exit $?" >> $OUT/pytest_golden.log
tail -3 $OUT/pytest_golden.log | cut -c1-500
P="BN=32,sk=4,tm=1 BN=32,sk=4,tm=1,cl=4 BN=32,sk=8,tm=1 BN=32,sk=8,tm=1,cl=4 BN=64,sk=4,tm=1 BN=64,sk=4,tm=1,cl=4 BN=32,sk=2,tm=1,cl=4"
timeout 300 python tools/try_params.py --ops 42:1,38:1,40:1,37:1,0:1,1:1,16:1,21:1,36:1,42:5,38:5 --params $P > $OUT/try.log 2>&1
P3="BN=32,sk=4,tm=3 BN=32,sk=4,tm=3,cl=4 BN=32,sk=8,tm=3,cl=4 BN=64,sk=2,tm=3,cl=4"
timeout 300 python tools/try_params.py --ops 3:1,4:1,7:1,8:1,11:1,3:5 --params $P3 > $OUT/try3.log 2>&1
PF="conv_fc:BN=32,sk=4,sw=1,tm=1 conv_fc:BN=32,sk=4,sw=1,tm=1,cl=4 conv_fc:BN=32,sk=8,sw=1,tm=1 conv_fc:BN=32,sk=8,sw=1,tm=1,cl=4"
timeout 300 python tools/try_params.py --ops 13:1,13:5,25:5,25:20 --params $PF > $OUT/tryfc.log 2>&1
cat $OUT/try.log $OUT/try3.log $OUT/tryfc.log | grep -v "^ \|Traceback\|File\|torch\.\|return"
