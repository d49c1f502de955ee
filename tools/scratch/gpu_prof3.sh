# launch list with per-kernel DRAM traffic (N=1 bench) + one --set full capture of the update / merge kernels
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --profile-phases 0 --cfg5 0"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_dram.csv $CMD > gpurun_out/ncu3.log 2>&1; echo rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_sgd_flat|k_sgd_single|MergeMap|k_grad_ptrs" -s 20 -c 8 -o gpurun_out/prof_r1_n1 $CMD > gpurun_out/ncu4.log 2>&1; echo rc=$?
