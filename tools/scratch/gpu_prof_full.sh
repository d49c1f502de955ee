# ncu --set full of the N=1 bench's top kernels (one capture per kernel name)
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --profile-phases 0 --cfg5 0"
$CMD > gpurun_out/plain.log 2>&1; echo plain rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_sgd_flat|k_sgd_single|k_copy_rows|k_radix_scatter}" -s ${SKIP:-60} -c ${COUNT:-6} -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_full.log
