# A/B: cfg2 bench with env A vs env B, alternated, same box
for i in 1 2; do
  env $A timeout 300 python bench.py --config ${CFG:-cfg2} --no-cpu-baseline > gpurun_out/ab_A$i.log 2>&1
  env $B timeout 300 python bench.py --config ${CFG:-cfg2} --no-cpu-baseline > gpurun_out/ab_B$i.log 2>&1
done
