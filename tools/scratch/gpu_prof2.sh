set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --profile-phases 0 --cfg5 0"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_sgd_flat|MergeMap|k_radix_scatter|k_sgd_combine" -s 16 -c 8 -o gpurun_out/prof_sgd $CMD > gpurun_out/ncu2.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu2.log
