#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list, ncu full captures
# of the dominant kernel and of the top TMA kernel.   usage (under gpurun): bash tools/gpu_round.sh TAG
set -x
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
cat $OUT/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch_bench.log 2>&1
ROW=$(python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['roofline']['corpus_row'])")
BATCH=$(python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['roofline']['op'].split(':in')[1].split('x')[0])")
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_(umma|tconv|tiled|simple|fc)" -s 2 -c 1 -o $OUT/prof_dom \
   python tools/run_op.py --row $ROW --batch $BATCH --reps 3 > $OUT/ncu_full.log 2>&1
if [ "$ROW" != "42" ] || [ "$BATCH" != "20" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_tconv" -s 2 -c 1 -o $OUT/prof_r42 \
   python tools/run_op.py --row 42 --batch 20 --reps 3 > $OUT/ncu_full42.log 2>&1
fi
du -sh $OUT/*
echo done
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "reference exit $?" >> $OUT/bench_reference.err
timeout 600 python bench.py --prec bf16 --no-cpu > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err
timeout 600 python tools/net_bench.py > $OUT/net_bench.jsonl 2> $OUT/net_bench.err
