# Round-2 final pass (bench lines, GPU suite, smoke, cfg2 launch list; no ncu --set full)
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg2_$TAG.log 2>&1; echo "bench cfg2 rc=$?"
for c in cfg1 cfg2u cfg2z12 cfg3 cfg4 cfg5 cfg5m; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --profile > gpurun_out/bench_${c}_$TAG.log 2>&1; echo "$c rc=$?"
done
timeout 600 python bench.py --config cfg4 --cache-partition --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg4p_$TAG.log 2>&1; echo "cfg4p rc=$?"
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_*.log')):
    try:
        d=json.loads([l for l in open(f) if l.startswith('{')][-1])
        print(f.split('/')[-1], round(d['ms_per_step']*1000,1), 'us', '%.3g' % d['value'], 'e2e %.3g' % (d['e2e']['value'] if isinstance(d.get('e2e'),dict) else 0), 'cpu', (d.get('cpu_baseline') or {}).get('value'))
    except Exception as e: print(f, 'ERR', e)
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_cfg2_$TAG.csv | tail -10
