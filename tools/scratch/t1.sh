export FSX_HUB_TIMEOUT_S=60
timeout 900 python -m pytest tests/test_gpu_parity_pinned.py -k "cfg4" -q -m gpu > gpurun_out/t1.log 2>&1; tail -5 gpurun_out/t1.log
grep -E "Error|error" gpurun_out/t1.log | head -5
