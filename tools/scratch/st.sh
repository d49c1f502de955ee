for v in "FSX_SPLIT_LANE=1" ; do
env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tests/mp_stress_direct.py 12 3 > gpurun_out/st.log 2>&1
echo "$v rc=$?"; grep -E "stress|STRESS|Error" gpurun_out/st.log | head -5 | cut -c1-250
done
