#!/bin/bash
# The non-headline configs on the current code: one bench line each (with the
# CPU reference leg) plus ncu launch lists for the cache and collection steps.
TAG=${1:-r1}
mkdir -p gpurun_out
for c in cfg1 cfg2u cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_${c}_$TAG.log 2>&1
  echo "$c rc=$?"
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_${c}_$TAG.log') if l.startswith('{')][-1]); print('$c', d['value'], d['ms_per_step'], d.get('cache'), d['e2e']['value'] if isinstance(d.get('e2e'), dict) else None)" || tail -5 gpurun_out/bench_${c}_$TAG.log
done
for c in cfg4 cfg5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${c}_$TAG.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "ncu $c rc=$?"
done
