mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_cache_fast_gpu.py -x -q > gpurun_out/pt_it9.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_it9.log
for i in 1 2; do for c in cfg2 cfg4 cfg2u; do
timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_it9.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_it9.log') if l.startswith('{')][-1]); print('$c', round(d['ms_per_step']*1000,1),'us')"
done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_it9.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_it9.csv | tail -8
