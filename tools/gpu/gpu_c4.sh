timeout 600 python -m pytest tests/test_cache_gpu.py -q -x > gpurun_out/pt_c4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_c4.log
timeout 400 python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo "cfg4 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg4.log').readline()); print(d['value'], d['ms_per_step'], d['cache'], d['e2e']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; python tools/launches.py gpurun_out/launches_cfg4.csv | grep -E "lfu|Radix|lookup"
