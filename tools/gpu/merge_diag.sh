mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "merge_units or planned_ranges or cfg2_full or fused_sgd" > gpurun_out/pytest_merge.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_merge.log
for v in 1 0; do
  TTGPU_MERGE1=$v TTGPU_LIB=$PWD/paper_2101_11714_b200/lib/libttgpu_diag.so timeout 400 python bench.py --config cfg2 --steps 10 --warmup 5 --no-cpu-baseline --cta-times gpurun_out/cta_m$v.npz > gpurun_out/bench_cta_m$v.log 2>&1
  echo "merge=$v rc=$?"; python tools/cta_marks.py gpurun_out/cta_m$v.npz 2>&1 | head -40
done
