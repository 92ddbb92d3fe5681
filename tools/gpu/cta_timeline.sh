# Per-CTA timelines of the fast-path kernels (diagnostics build, bench.py --cta-times)
mkdir -p gpurun_out
make lib-diag > /dev/null 2>&1 || true
for c in ${CONFIGS:-cfg2 cfg2u}; do
  TTGPU_LIB=$PWD/paper_2101_11714_b200/lib/libttgpu_diag.so timeout 400 python bench.py --config $c --steps 10 --warmup 5 --no-cpu-baseline --cta-times gpurun_out/cta_$c.npz > gpurun_out/bench_cta_$c.log 2>&1
  echo "$c rc=$?"; python tools/cta_marks.py gpurun_out/cta_$c.npz
done
