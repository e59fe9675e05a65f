#!/bin/bash
# r2ak: first-layer space-to-depth (tm=6): parity + timings vs the x-window path
OUT=gpurun_out/r2ak; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or space_to_depth" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log | cut -c1-400
P="BN=96,sk=1,tm=1 BN=96,sk=1,tm=6 BN=96,sk=1,tm=6,cl=3 BN=64,sk=1,tm=1,oc=2 BN=64,sk=1,tm=6,oc=2"
timeout 400 python tools/try_params.py --ops 34:20,33:20,35:20,34:5,35:5,34:1 --params $P > $OUT/try.log 2>&1
cat $OUT/try.log | grep -v "^ \|Traceback\|File\|torch\.\|return" | awk '{print $1,$2,$3,$4,$5,$7,$9,$10}'
