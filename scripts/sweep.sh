#!/bin/bash
# Bench sweep (GPU box).  usage: scripts/sweep.sh OUT "ENV=.. ENV2=.. | --bench-args" ...
out=$1; shift
for cfg in "$@"; do
  envs="${cfg%%|*}"; args="${cfg#*|}"; [ "$args" = "$cfg" ] && args=""
  echo "== $cfg" >> "$out"
  env $envs python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $args 2>&1 | tail -1 | \
    python -c "import sys,json
l=sys.stdin.read()
try:
  d=json.loads(l); r=d['roofline']; print(d['value'], d['ms_per_step'], r['iteration']['frac'], r['kernels_ms_per_iter'], d['setup_s'])
except Exception: print('FAIL', l[-600:])" >> "$out"
done
