mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"f3_srows|f3_bwd1" -s 10 -c 2 -o gpurun_out/srows python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_srows.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_srows.log
