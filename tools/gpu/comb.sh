mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_cache_fast_gpu.py -m gpu -x -q > gpurun_out/pytest_comb.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_comb.log
for c in cfg2 cfg2u cfg4; do
  TTGPU_LIB=$PWD/paper_2101_11714_b200/lib/libttgpu_diag.so timeout 400 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --cta-times gpurun_out/cta5_$c.npz > gpurun_out/bench_cta5_$c.log 2>&1
  echo "$c rc=$?"; python tools/cta_marks.py gpurun_out/cta5_$c.npz | grep -A2 combine; grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_cta5_$c.log
done
