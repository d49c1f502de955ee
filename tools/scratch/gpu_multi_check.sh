# multi-GPU check at HEAD: multi-process / balancer tests, bench at N = 2 and 4 (cfg5 included)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_balancer_ce.py -x -q 2>&1 | tail -3
NG=$(python -c "import torch; print(torch.cuda.device_count())")
for N in 2 4; do
  [ "$N" -le "$NG" ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo rc=$?
  python -c "
import json; d=json.loads(open('gpurun_out/bench_n$N.json').read().strip().splitlines()[-1]); print($N, d['value'], d['ms_per_step'], d['exposed_comm_ms_per_iter'], json.dumps(d.get('cfg5'))[:600])"
done
