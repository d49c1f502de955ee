# A/B on the N=1 bench phases. Each argument is a variant: a name `v` selects
# tools/variants/libfsx_v.so; `env:K=V,K2=V2` runs the in-tree library with
# those environment variables; `cur` the in-tree library as is.
for v in "$@"; do
  lib=""; envs=""
  case "$v" in
    env:*) envs=$(echo "${v#env:}" | tr ',' ' ');;
    cur) ;;
    *) lib="FSX_LIB=$PWD/tools/variants/libfsx_$v.so";;
  esac
  tag=$(echo "$v" | tr ':=,' '___')
  env $lib $envs timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --cfg5 0 ${AB_ARGS:-} > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$tag.json').read().strip().splitlines()[-1]); ph=d['phases_ms_per_step']
print('$v', round(d['value']/1e6,1), 'Mrows/s', d['ms_per_step'], ph)"
done
