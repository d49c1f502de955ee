out=gpurun_out/mb; mkdir -p $out
for n in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n --steps 20 --warmup 5 > $out/bench_n$n.json 2> $out/bench_n$n.err
echo "n=$n rc=$?"
done
