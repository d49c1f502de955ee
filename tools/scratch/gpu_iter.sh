# quick iteration: engine parity tests, A/B of variants on the N=1 bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_primitives.py -x -q 2>&1 | tail -4
bash tools/ab.sh "$@"
