set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo pytest=$? >> gpurun_out/r2a_pytest.log
for c in cfg2 cfg3 cfg4; do timeout 400 python bench.py --config $c --profile > gpurun_out/r2a_bench_$c.log 2>&1; done
tail -3 gpurun_out/r2a_pytest.log
