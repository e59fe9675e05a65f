set -x
OUT=gpurun_out/r2a; mkdir -p $OUT
nvidia-smi -L > $OUT/smi.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for S in 1 2 4 8; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --streams $S > $OUT/bench_s$S.json 2> $OUT/bench_s$S.err
  B2C_NO_PDL=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --streams $S > $OUT/bench_s${S}_nopdl.json 2> $OUT/bench_s${S}_nopdl.err
done
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_signed_sweep.py tests/test_reference_dropin.py -x -q -m gpu > $OUT/pytest_new.log 2>&1; echo "exit $?" >> $OUT/pytest_new.log
tail -5 $OUT/pytest_new.log
for f in $OUT/bench_s*.json; do echo $f; python -c "import json,sys;d=json.load(open('$f'));print(d['value'],d['ms_per_step'],d['config']['group_ms'],d['config']['serial_ms_per_step_rank0'],d['clocks'])"; done
