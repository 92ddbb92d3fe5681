mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wide3_gpu.py tests/test_fullsize_gpu.py tests/test_parity_gpu.py -x -q -k "wide3 or cfg3 or random or f64 or golden" > gpurun_out/pt_it10.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_it10.log
for i in 1 2; do timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --profile --no-cpu-baseline > gpurun_out/bench_it10.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_it10.log') if l.startswith('{')][-1]); print('cfg3', round(d['ms_per_step']*1000,1),'us', json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))"; done
