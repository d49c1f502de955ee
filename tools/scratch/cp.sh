set -x
mkdir -p gpurun_out/cp
timeout 900 python -m pytest tests/test_gpu_parity_pinned.py tests/test_gpu_engine.py -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/chain_profile.py 4 8 0 > gpurun_out/cp/run.txt 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cp/launches2.csv python tools/chain_profile.py 4 8 0 > gpurun_out/cp/ncu1.txt 2>&1
