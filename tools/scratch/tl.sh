set -x
mkdir -p gpurun_out/tl
python -m pytest tests/test_gpu_parity_pinned.py -k cfg4 tests/test_gpu_multiproc.py -x -q -m gpu 2>&1 | tail -5
for n in 4; do for v in 1; do
FSX_COG_DIRECT=1 FSX_ECO_DIRECT=1 FSX_TRACE_COPIES=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 tools/timeline.py --victim $v --iters 10 --profile-from 6 > gpurun_out/tl/sum_n${n}_v${v}_dd.txt 2>&1
mkdir -p gpurun_out/tl/n${n}_v${v}_dd; mv gpurun_out/timeline_r*.txt gpurun_out/tl/n${n}_v${v}_dd/
done; done
