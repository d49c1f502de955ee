set -x
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_multiproc.py -x -q 2>&1 | tail -3
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/timeline.py --victim 1 --presum 1 2>&1 | grep -v Warning | tail -8
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_n4.json').read().strip().splitlines()[-1]); print(d['value'], d['exposed_comm_ms_per_iter'], json.dumps(d['cfg5']))"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'], d['phases_ms_per_step'])"
