OUT=gpurun_out/multi
mkdir -p $OUT
export B2C_BENCH_ONE_GPU_TEST=1
for mode in "" "--strong" "--gather"; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-e2e $mode > $OUT/bench2$mode.json 2> $OUT/bench2$mode.err; echo "exit $? $mode"; head -c 400 $OUT/bench2$mode.json; echo; tail -3 $OUT/bench2$mode.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err; echo "ref exit $?"; head -c 600 $OUT/ref.json; echo
