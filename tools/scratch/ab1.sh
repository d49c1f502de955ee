for r in 1 2; do
tools/ab_env.sh gpurun_out/ab "FSX_STREAM_VARIANT=0" "FSX_STREAM_VARIANT=4" "FSX_STREAM_VARIANT=1"
done
