mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bench_pooling.py tests/test_streams_gpu.py tests/test_checkpoint.py -q -s > gpurun_out/pytest_cov2.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_cov2.log
timeout 600 python -m paper_2101_11714_b200.bench_pooling --rows 100000 --ranks 8 16 32 64 --poolings 1 10 100 --bags 256 --reps 30 --out gpurun_out/bench_pooling_default.csv; echo "sweep rc=$?"; cat gpurun_out/bench_pooling_default.csv
