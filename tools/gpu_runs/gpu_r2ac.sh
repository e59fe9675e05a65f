#!/bin/bash
# r2ac: bf16 SS path (tm=5, MODE 8): parity + timings vs the TS path
OUT=gpurun_out/r2ac; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_bf16_gpu.py -q -x > $OUT/pytest_bf16.log 2>&1; echo "exit $?" >> $OUT/pytest_bf16.log
tail -15 $OUT/pytest_bf16.log | cut -c1-400
P="BN=128,sk=0,tm=1,pr=1 BN=128,sk=1,tm=1,pr=1 BN=128,sk=0,tm=5,pr=1 BN=128,sk=1,tm=5,pr=1 BN=192,sk=0,tm=5,pr=1 BN=64,sk=1,tm=5,pr=1"
timeout 400 python tools/try_params.py --ops 42:20,41:20,40:20,39:20,38:20,29:20,27:20,6:20,42:5,40:5,38:1,3:1 --params $P > $OUT/try.log 2>&1
cat $OUT/try.log | grep -v "^ \|Traceback\|File\|torch\.\|return" | awk '{print $1,$2,$3,$4,$5,$7,$9,$10}'
