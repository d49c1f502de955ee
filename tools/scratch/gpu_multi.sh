# N>1 bench lines (+ a timeline of rank spans); usage: bash tools/gpu_multi.sh N
set -x
N=${1:-2}
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_n$N.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], 'host', d.get('host_enqueue_ms_per_step'), 'exp', d['exposed_comm_ms_per_iter']); print(d['phases_ms_per_step']); print(json.dumps(d['cfg5']))"
if [ "${TIMELINE:-1}" = 1 ]; then
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tools/timeline.py --victim 0 --presum 1 --iters 10 --profile-from 7 2>&1 | grep "^rank" | tail -8
fi
