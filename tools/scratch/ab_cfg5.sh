# A/B of environment variants on the config-5 line at N GPUs:
#   bash tools/ab_cfg5.sh N "FSX_PDL=0" "FSX_PDL=1" ...
N=$1; shift
mkdir -p gpurun_out
k=0
for v in "$@"; do
  k=$((k+1))
  env $v timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700+k)) bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/ab5_${N}_$k.json 2> gpurun_out/ab5_${N}_$k.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab5_${N}_$k.json').read().strip().splitlines()[-1]); c=d['cfg5']
print('$v', round(d['value']/1e6,1), 'Mrows/s', d['ms_per_step'], 'exp', d['exposed_comm_ms_per_iter'], 'cfg5', c['exposed_ms_per_iter_max_over_ranks'], c['exposed_reduction_pct'], c['step_ms'], c['victim_alone_ms'], c['victim_alone_ms_min_over_ranks'])"
done
