# Round evidence at N=1: default bench line, ncu launch list (time + DRAM bytes
# per launch), one ncu --set full capture of the top kernels.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench rc=$?
tail -1 gpurun_out/bench_n1.json
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --profile-phases 0 --cfg5 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sgd_warp|k_sgd_single|k_copy_rows|k_os_scatter|k_radix_scatter" -s 60 -c 8 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -2 gpurun_out/ncu_full.log
