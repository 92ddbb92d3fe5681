# per-kernel durations inside the bench (graph replays), warm caches, no clock lock
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -c ${COUNT:-200} --csv --log-file gpurun_out/${OUT:-launches}.csv python bench.py --config ${CFG:-cfg2} --steps 4 --warmup 3 --no-cpu-baseline $BENCH_ARGS > gpurun_out/${OUT:-launches}.log 2>&1
echo rc=$?
