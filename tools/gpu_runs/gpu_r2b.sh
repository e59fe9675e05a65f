# on-chip B lo: parity + bench A/B (groups, streams)
OUT=gpurun_out/r2b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for S in 4 8; do for G in one batch; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --streams $S --groups $G > $OUT/bench_s${S}_$G.json 2> $OUT/bench_s${S}_$G.err
done; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --streams 1 --groups one --per-op-out $OUT/per_op.csv > $OUT/bench_s1.json 2> $OUT/bench_s1.err
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
for f in $OUT/bench_s*.json; do echo $f; python -c "import json,sys;d=json.load(open('$f'));print(d['value'],d['ms_per_step'],d['config']['group_ms'],d['config']['serial_ms_per_step_rank0'],d['clocks']['sm_mhz'], d['roofline']['frac_of_mode_peak'])"; done
