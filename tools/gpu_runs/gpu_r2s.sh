#!/bin/bash
# r2p: Winograd F(2x2,3x3) parity + timings vs the direct tcgen05 kernels
OUT=gpurun_out/r2s; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k golden > $OUT/pytest_golden.log 2>&1; echo "exit $?" >> $OUT/pytest_golden.log
tail -25 $OUT/pytest_golden.log | cut -c1-600
P="BN=128,sk=0,tm=1 BN=128,sk=0,tm=1,cl=3 conv_wino:BN=128,sk=1,tm=1 conv_wino:BN=192,sk=1,tm=1 conv_wino:BN=64,sk=1,tm=1 conv_wino:BN=128,sk=0,tm=1 conv_wino:BN=128,sk=1,sw=1,tm=1 conv_wino:BN=192,sk=0,sw=1,tm=1"
timeout 400 python tools/try_params.py --ops 40:20,37:20,38:20,36:20,39:20,32:20,28:20,22:20,16:20,40:5,38:5,36:5,32:5,40:1,38:1 --params $P > $OUT/try.log 2>&1
cat $OUT/try.log
