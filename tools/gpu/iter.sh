# quick iteration: selected GPU tests + cfg2 bench with per-phase profile
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTS:-cluster_sort or fast_path or cfg2 or fused_device}" > gpurun_out/iter_pytest.log 2>&1; echo pytest=$? >> gpurun_out/iter_pytest.log
tail -3 gpurun_out/iter_pytest.log
for c in ${CFGS:-cfg2}; do timeout 300 python bench.py --config $c --profile --no-cpu-baseline $BENCH_ARGS > gpurun_out/iter_bench_$c.log 2>&1; done
