# cache fast path + wide3 iteration: targeted GPU tests, then cfg3 / cfg4 / cfg2z12 bench lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cache_fast_gpu.py tests/test_wide3_gpu.py tests/test_cache_gpu.py -x -q > gpurun_out/pt_it2.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_it2.log
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_parity_gpu.py -x -q -k "cfg3 or cfg4" > gpurun_out/pt_it2_full.log 2>&1; echo "pytest full rc=$?"; tail -8 gpurun_out/pt_it2_full.log
for a in "--config cfg3" "--config cfg4" "--config cfg2z12"; do
  timeout 600 python bench.py $a --steps 10 --warmup 5 --profile --no-cpu-baseline > gpurun_out/bench_it2.log 2>&1; echo "bench $a rc=$?"
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_it2.log') if l.startswith('{')][-1]); print(round(d['ms_per_step']*1000,1),'us', d['value'], 'e2e', d['e2e']['value'], d.get('cache'), json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))" || tail -20 gpurun_out/bench_it2.log
done
