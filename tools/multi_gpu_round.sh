#!/bin/bash
# Multi-GPU evidence on one box (gpurun --gpus N): multi-process parity tests,
# then bench lines at N=2 and N=4 (torchrun, one rank per GPU) with the
# config-5 section (blocking NCCL vs prioritized copy-engine, SM contention).
# usage: tools/multi_gpu_round.sh OUTDIR
out=${1:-gpurun_out/multi}
mkdir -p "$out"
ng=$(python -c "import torch;print(torch.cuda.device_count())")
echo "gpus: $ng" | tee "$out/info.txt"
nvidia-smi topo -m > "$out/topo.txt" 2>&1
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_balancer_ce.py -q -s -p no:cacheprovider \
  > "$out/pytest_multi.log" 2>&1; echo "pytest rc=$?" | tee -a "$out/info.txt"
for n in 2 4; do
  [ "$n" -le "$ng" ] || continue
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n --steps 20 --warmup 5 \
    > "$out/bench_n$n.json" 2> "$out/bench_n$n.err"
  echo "bench n=$n rc=$?" | tee -a "$out/info.txt"
  grep -a "nChannels\|Channel [0-9]*/[0-9]* :" "$out/bench_n$n.err" | head -20 > "$out/nccl_channels_n$n.txt"
done
