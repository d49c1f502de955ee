set -x
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -15
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo rc=$?
tail -c 3000 gpurun_out/bench_n$N.json
done
