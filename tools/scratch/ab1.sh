set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python -m pytest tests/test_gpu_engine.py tests/test_gpu_primitives.py -x -q -m gpu 2>&1 | tail -3
for r in 1 2; do
tools/ab_env.sh gpurun_out/ab "FSX_LIB=tools/variants/libfsx_p8.so" "FSX_LIB=paper_2604_24073_b200/libfsx.so" "FSX_LIB=tools/variants/libfsx_i4.so" "FSX_LIB=tools/variants/libfsx_i2.so"
done
