export FSX_HUB_TIMEOUT_S=30
timeout 1100 python -m pytest tests/test_gpu_engine.py tests/test_gpu_multiproc.py tests/test_gpu_pooled.py tests/test_gpu_pipeline.py tests/test_gpu_parity_pinned.py -q -m gpu > gpurun_out/t1.log 2>&1
tail -5 gpurun_out/t1.log
