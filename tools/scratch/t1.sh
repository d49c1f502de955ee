cd paper_2604_24073_b200/cpp
CUDA_MODULE_LOADING=EAGER timeout 120 ./build/ref_test_pipeline "-tce=balancer communication is fully overlapped*" 2>&1 | tail -2
