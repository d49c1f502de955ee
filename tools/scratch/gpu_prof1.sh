set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --profile-phases 0"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sgd_chunks|k_copy_rows|k_radix_scatter|k_co_apply" -s 200 -c 8 -o gpurun_out/prof_n1 $CMD > gpurun_out/ncu2.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu2.log
