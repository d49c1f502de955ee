out=gpurun_out/mb3; mkdir -p $out
export FSX_HUB_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity_pinned.py tests/test_gpu_multiproc.py -x -q -m gpu > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for n in 4 2; do
for sl in 1 0; do
FSX_SPLIT_LANE=$sl timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n --steps 20 --warmup 5 --cfg5 0 > $out/bench_n${n}_$sl.json 2> $out/bench_n${n}_$sl.err
python -c "import json;d=json.loads(open('$out/bench_n${n}_$sl.json').read().strip().splitlines()[-1]);print('$n split=$sl', d['value'], d['ms_per_step'], d['host_enqueue_ms_per_step'], d['exposed_comm_ms_per_iter'], d['e2e']['value'])"
done; done
for sl in 1 0; do FSX_SPLIT_LANE=$sl timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_n1_$sl.json 2>/dev/null; python -c "import json;d=json.loads(open('$out/bench_n1_$sl.json').read().strip().splitlines()[-1]);print('1 split=$sl', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"; done
