#!/bin/bash
# r2ag: two loader warps (pixels | filters): parity + timings
OUT=gpurun_out/r2ag; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bf16_gpu.py tests/test_fp8_gpu.py -q -x -k "golden or split_k or slabs or signed or full_size" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log | cut -c1-400
P="BN=128,sk=1,tm=5,pr=1 BN=128,sk=1,tm=5,cl=3,pr=1 BN=192,sk=1,tm=5,cl=3,pr=1 BN=128,sk=0,tm=5,cl=3,pr=1 BN=192,sk=0,tm=5,cl=3,pr=1"
timeout 400 python tools/try_params.py --ops 42:20,41:20,40:20,39:20,38:20,37:20,36:20,42:5,6:20 --params $P > $OUT/try.log 2>&1
cat $OUT/try.log | grep -v "^ \|Traceback\|File\|torch\.\|return" | awk '{print $1,$2,$3,$4,$5,$7,$9,$10}'
B="MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1"
timeout 60 python tools/trace_op.py --row 42 --batch 20 --params "$B,BN=128,sk=1,sw=0,dr=0,tm=5,pr=1" 2>&1 | sed -n 1,9p | cut -c1-300
