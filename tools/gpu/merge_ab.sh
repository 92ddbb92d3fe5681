# merge units: parity subset, A/B vs libttgpu_base.so, and the cfg2 per-CTA timeline
CONFIGS="${CONFIGS:-cfg2 cfg4 cfg2z12}" bash tools/gpu/ab_lib.sh
for v in 1 0; do
  TTGPU_MERGE1=$v TTGPU_LIB=$PWD/paper_2101_11714_b200/lib/libttgpu_diag.so timeout 400 python bench.py --config cfg2 --steps 10 --warmup 5 --no-cpu-baseline --cta-times gpurun_out/cta_m$v.npz > gpurun_out/bench_cta_m$v.log 2>&1
  echo "merge=$v rc=$?"; python tools/cta_marks.py gpurun_out/cta_m$v.npz 2>&1 | grep -A1 "f3_srows_bwd2\|f3_bwd1 "
done
