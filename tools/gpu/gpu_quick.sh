mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_q.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_q.log').readline()); print(d['value'], d['ms_per_step'], d['e2e'], d['phases_ms'])"
