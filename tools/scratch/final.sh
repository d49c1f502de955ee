timeout 420 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/final_pytest.log
