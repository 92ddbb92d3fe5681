mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cache_fast_gpu.py tests/test_cache_gpu.py tests/test_sanitizer_gpu.py -x -q > gpurun_out/pt_it6.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pt_it6.log
timeout 600 python -m pytest tests/test_fullsize_gpu.py -x -q -k cfg4 > gpurun_out/pt_it6f.log 2>&1; echo "pytest full rc=$?"; tail -2 gpurun_out/pt_it6f.log
for a in "--config cfg4" "--config cfg2z12" "--config cfg3"; do
timeout 300 python bench.py $a --steps 20 --warmup 5 --profile --no-cpu-baseline > gpurun_out/bench_it6.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_it6.log') if l.startswith('{')][-1]); print('$a', round(d['ms_per_step']*1000,1),'us', json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))" || tail -5 gpurun_out/bench_it6.log
done
