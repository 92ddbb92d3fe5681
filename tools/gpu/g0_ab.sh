# f3_combine dG0 group size (kGroup0) variants: parity subset per library, then timing
mkdir -p gpurun_out
for v in g64 g128; do
  TTGPU_LIB=$PWD/paper_2101_11714_b200/lib/libttgpu_$v.so timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_cache_fast_gpu.py -m gpu -q -x > gpurun_out/pytest_$v.log 2>&1
  echo "$v pytest rc=$?"; tail -1 gpurun_out/pytest_$v.log
done
VARIANTS="g32 g64 g128" CONFIGS="cfg2 cfg2z12 cfg4" bash tools/gpu/ab_multi.sh
