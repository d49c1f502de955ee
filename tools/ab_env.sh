#!/bin/bash
# A/B of engine tuning knobs on one GPU: each argument is a list of env
# assignments and/or bench.py flags ("FSX_STREAM_VARIANT=2 --reduce-chunk 32");
# prints step, update launch time, roofline fraction and side-lane phases of
# `python bench.py` under each.
# usage (on the GPU box): tools/ab_env.sh OUTDIR "CFG..." "CFG..." ...
out=$1; shift
mkdir -p "$out"
for cfg in "$@"; do
  envs=(); args=()
  for tok in $cfg; do
    if [[ $tok == *=* && $tok != -* ]]; then envs+=("$tok"); else args+=("$tok"); fi
  done
  env "${envs[@]}" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "${args[@]}" > "$out/b.json" 2>>"$out/ab.err"
  python -c "import json,sys;d=json.load(open('$out/b.json'));p=d['phases_ms_per_step'];print('$cfg |', d['ms_per_step'], d['roofline']['launch_ms'], d['roofline']['frac'], 'merge', p.get('merge'), 'collide', p.get('collide'), 'dedup', p.get('dedup'), 'exposed', p.get('exposed'))"
done
