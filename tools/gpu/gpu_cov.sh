mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_cov.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_cov.log
timeout 400 python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo "cfg4 rc=$?"; tail -c 1500 gpurun_out/bench_cfg4.log
