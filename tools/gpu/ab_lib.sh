# A/B of two library builds (TTGPU_LIB): base = HEAD, new = working tree; alternating runs.
# base: git stash; make lib; cp paper_2101_11714_b200/lib/libttgpu.so paper_2101_11714_b200/lib/libttgpu_base.so; git stash pop; make lib
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_cache_fast_gpu.py -m gpu -x -q > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ab.log
for c in ${CONFIGS:-cfg2 cfg2u cfg4}; do
  for rep in 1 2 3; do
    for v in base new; do
      if [ $v = base ]; then L=paper_2101_11714_b200/lib/libttgpu_base.so; else L=paper_2101_11714_b200/lib/libttgpu.so; fi
      TTGPU_LIB=$PWD/$L timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${c}_${v}_$rep.log 2>&1
      echo "$c $v $rep $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${c}_${v}_$rep.log)"
    done
  done
done
