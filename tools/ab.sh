# A/B the libfsx variants in tools/variants on the N=1 bench phases
for v in "$@"; do
  FSX_LIB=$PWD/tools/variants/libfsx_$v.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --cfg5 0 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); ph=d['phases_ms_per_step']
print('$v', round(d['value']/1e6,1), 'Mrows/s', d['ms_per_step'], {k: ph[k] for k in ('merge','split','co_update','ex_update','dedup','exposed') if k in ph})"
done
