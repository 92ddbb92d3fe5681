# Round-2 re-entry pass: full GPU suite, smoke, bench lines for cfg2/cfg2u/cfg3/cfg4, cfg2 launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_r2c.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2c.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_r2c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2c.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_r2c.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg2_r2c.log 2>&1; echo "bench rc=$?"; head -c 3000 gpurun_out/bench_cfg2_r2c.log
for c in cfg2u cfg3 cfg4; do timeout 600 python bench.py --config $c --steps 10 --warmup 5 --profile --no-cpu-baseline > gpurun_out/bench_${c}_r2c.log 2>&1; echo "$c rc=$?"; head -c 1500 gpurun_out/bench_${c}_r2c.log; echo; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2c.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_r2c.csv | tail -20
