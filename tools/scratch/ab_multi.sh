# A/B of environment variants at N GPUs: bash tools/ab_multi.sh N "FSX_ONESWEEP=1" "FSX_ONESWEEP=0" ...
N=$1; shift
mkdir -p gpurun_out
k=0
for v in "$@"; do
  k=$((k+1))
  env $v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+k)) bench.py --gpus $N --steps 10 --warmup 3 --cfg5 0 > gpurun_out/abm_$k.json 2> gpurun_out/abm_$k.err
  python -c "
import json; d=json.loads(open('gpurun_out/abm_$k.json').read().strip().splitlines()[-1])
print('$v', round(d['value']/1e6,1), 'Mrows/s', d['ms_per_step'], 'exp', d['exposed_comm_ms_per_iter'], {k: v for k, v in d['phases_ms_per_step'].items() if k in ('dedup','route','masks','split','collide','merge')})"
done
