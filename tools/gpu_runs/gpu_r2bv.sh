#!/bin/bash
# r2bv: final validation of the round-2 tree (BN=16 fc tile, shipped DBs): pytest -m gpu, smoke, sanitizers, benches (fp32 / bf16 / fp8 / reference arm), ncu launch list + full captures
OUT=gpurun_out/r2bv; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -5 $OUT/build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log; tail -1 $OUT/smoke.log
timeout 300 python tools/sanitize_ops.py > $OUT/sanitize_plain.log 2>&1; echo "exit $?" >> $OUT/sanitize_plain.log; tail -2 $OUT/sanitize_plain.log
for T in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_ops.py > $OUT/sanitize_$T.log 2>&1; echo "exit $?" >> $OUT/sanitize_$T.log
  echo "$T: $(grep -E 'ERROR SUMMARY|sanitize_ops:' $OUT/sanitize_$T.log | tr '\n' ' ') $(tail -1 $OUT/sanitize_$T.log)"
done
timeout 900 python bench.py --per-op-out $OUT/per_op.csv > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));c=d['config'];print('fp32',d['value'],d['ms_per_step'],c['per_batch_ms_isolated'],c['per_batch_ms_back_to_back'],d['roofline']['achieved'],d['roofline']['frac_of_mode_peak'],d['e2e']['value'],d['e2e']['frac_of_copy_bound'],d['cpu_baseline']['value'],d['clocks'])"
timeout 600 python bench.py --prec bf16 --no-cpu --no-e2e --per-op-out $OUT/per_op_bf16.csv > $OUT/bench_bf16.json 2> $OUT/bench_bf16.err
timeout 600 python bench.py --prec fp8 --no-cpu --no-e2e --per-op-out $OUT/per_op_fp8.csv > $OUT/bench_fp8.json 2> $OUT/bench_fp8.err
python -c "import json;[print(n,json.load(open(f'$OUT/bench_{n}.json'))['value']) for n in ('bf16','fp8')]"
timeout 1200 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
python -c "import json;d=json.load(open('$OUT/bench_reference.json'));print('reference',d['value'],d['ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $OUT/ncu_launch.log 2>&1
python tools/ncu_summary.py --launches $OUT/launches.csv > $OUT/launches.md 2>&1; head -12 $OUT/launches.md
cap() {  # name row batch kernel-regex [run_op args]
  local name=$1 row=$2 batch=$3 kre=$4; shift 4
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 -o $OUT/$name \
     python tools/run_op.py --row $row --batch $batch --reps 3 "$@" > $OUT/$name.log 2>&1
  echo "$name: $(tail -1 $OUT/$name.log)"
}
cap dom_r42n20 42 20 "k_tconv"
cap fcb_r13n5 13 5 "k_fc_bulk" --variant conv_fc_stream --params "MNt=1:1,MNb=8:1,Kb=3,vw=1,lf=1,li=1"
cap fcs_r25n1 25 1 "k_fc_stream"
cap first_r35n20 35 20 "k_tconv"
python tools/ncu_summary.py $(for f in $OUT/*.ncu-rep; do echo --rep $f; done) > $OUT/ncu_summary.md 2>&1
cat $OUT/ncu_summary.md | head -20
ncu -i $OUT/dom_r42n20.ncu-rep --page raw --csv > $OUT/dom_r42n20.raw.csv 2>/dev/null
find $OUT -name "*.ncu-rep" ! -name "dom_r42n20.ncu-rep" -delete
