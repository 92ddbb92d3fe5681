# ncu --set full of f3_bwd1 / f3_combine / f3_fwd (source-level, for tools/srcprof.py).
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"f3_bwd1|f3_combine|f3_fwd" -s 6 -c 3 -o gpurun_out/bwd1b python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_b.log
