mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_collection_gpu.py -q -x > gpurun_out/pt_col.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_col.log
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.log 2>&1; echo "cfg5 rc=$?"; tail -c 1500 gpurun_out/bench_cfg5.log
