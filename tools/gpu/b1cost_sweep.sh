# f3_bwd1 merge-unit range weights (TTGPU_B1COST=tile,cont): cfg2 / cfg2z12 / cfg4 step time, alternating
mkdir -p gpurun_out
for rep in 1 2; do
  for w in ${WS:-4,1 6,1 8,1 4,0 6,2 10,1 3,1}; do
    for c in cfg2 cfg2z12 cfg4; do
      TTGPU_B1COST=$w timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/sw_${c}_${w}_$rep.log 2>&1
      echo "$c w=$w rep=$rep $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/sw_${c}_${w}_$rep.log)"
    done
  done
done
