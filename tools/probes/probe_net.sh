OUT=gpurun_out/net1
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_net_gpu.py -x -q -m gpu > $OUT/pytest_net.log 2>&1; tail -3 $OUT/pytest_net.log
timeout 600 python tools/net_bench.py > $OUT/net_bench.jsonl 2> $OUT/net_bench.err; cat $OUT/net_bench.jsonl; tail -3 $OUT/net_bench.err
