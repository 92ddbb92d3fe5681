mkdir -p gpurun_out
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/e2e_probe.log | tail -12
for c in cfg1 cfg2u cfg3; do
timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$c.log').readline()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['phases_ms'])" 2>&1 | tail -3
done
