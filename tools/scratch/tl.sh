mkdir -p gpurun_out/tl3
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tools/timeline.py --victim 0 --iters 12 --profile-from 8 > gpurun_out/tl3/sum.txt 2>&1
mv gpurun_out/timeline_r*.txt gpurun_out/tl3/
