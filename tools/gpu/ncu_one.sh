# ncu --set full (source-level) of the kernels matching $KREGEX in a short cfg2 bench run
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${KREGEX}" -s ${SKIP:-6} -c ${COUNT:-1} -o gpurun_out/${OUT:-one} python bench.py --config ${CFG:-cfg2} --steps 2 --warmup 3 --no-cpu-baseline $BENCH_ARGS > gpurun_out/ncu_one.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_one.log
