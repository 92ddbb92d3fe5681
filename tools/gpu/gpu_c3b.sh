timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_cache_gpu.py -q -x > gpurun_out/pt_c3b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_c3b.log
timeout 400 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg3.log').readline()); print(d['value'], d['ms_per_step'], d['phases_ms'])"
