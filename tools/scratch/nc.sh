mkdir -p gpurun_out/nc
for n in 2 4; do
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,COLL timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29544 tools/nccl_ce_compare.py 8 > gpurun_out/nc/n$n.json 2> gpurun_out/nc/n$n.err
echo "n=$n rc=$?"; grep "^{" gpurun_out/nc/n$n.json
done
