# Round-2 evidence pass: full GPU suite, smoke, every config's bench line, cfg2 launch list + ncu
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
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum --clock-control none -k regex:f3_ -c 60 --csv --log-file gpurun_out/kern_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_kernels.py gpurun_out/kern_$TAG.csv cfg2 gpurun_out/ncu_kernels_$TAG.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:f3_ -s 30 -c 6 -o gpurun_out/full_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncufull_$TAG.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_w3|k_head|f3_gsort" -s 4 -c 6 -o gpurun_out/full3_$TAG python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncufull3_$TAG.log 2>&1; echo "ncu full3 rc=$?"
