out=gpurun_out/hang2; mkdir -p $out
for k in 1 2 3; do
setsid timeout -s KILL 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + k)) bench.py --gpus 4 --steps 20 --warmup 5 --cfg5 0 > $out/b.json 2> $out/b.err
rc=$?
echo "run $k rc=$rc $(python -c "import json;d=json.loads(open('$out/b.json').read().strip().splitlines()[-1]);print(d['ms_per_step'])" 2>/dev/null)"
nvidia-smi --query-compute-apps=pid --format=csv,noheader | head -3
done
