# cache fast path: cache + fullsize + parity GPU tests, cfg4 (fast / partition) and cfg2z12 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cache_fast_gpu.py tests/test_cache_gpu.py -x -q > gpurun_out/pt_cache.log 2>&1; echo "pytest cache rc=$?"; tail -15 gpurun_out/pt_cache.log
timeout 900 python -m pytest tests/test_fullsize_gpu.py -x -q -k cfg4 > gpurun_out/pt_cache_full.log 2>&1; echo "pytest full rc=$?"; tail -5 gpurun_out/pt_cache_full.log
for a in "--config cfg4" "--config cfg4 --cache-partition" "--config cfg2z12"; do
  timeout 600 python bench.py $a --steps 20 --warmup 5 --profile --no-cpu-baseline > gpurun_out/bench_cache.log 2>&1; echo "bench $a rc=$?"
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_cache.log') if l.startswith('{')][-1]); print(round(d['ms_per_step']*1000,1),'us', d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step_median'], d.get('cache'), d['execution']['graph'], json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))" || tail -20 gpurun_out/bench_cache.log
done
