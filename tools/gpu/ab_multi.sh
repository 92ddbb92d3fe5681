# A/B/C of library builds (TTGPU_LIB): libttgpu.so vs libttgpu_<v>.so for v in $VARIANTS, alternating
mkdir -p gpurun_out
for c in ${CONFIGS:-cfg2 cfg2z12}; do
  for rep in 1 2 3; do
    for v in base ${VARIANTS}; do
      if [ $v = base ]; then L=paper_2101_11714_b200/lib/libttgpu.so; else L=paper_2101_11714_b200/lib/libttgpu_$v.so; fi
      TTGPU_LIB=$PWD/$L timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abm_${c}_${v}_$rep.log 2>&1
      echo "$c $v $rep $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/abm_${c}_${v}_$rep.log)"
    done
  done
done
