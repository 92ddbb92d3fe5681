# quick cfg2/cfg4 timing (3 alternating runs)
for i in 1 2 3; do for c in cfg2 cfg4; do
timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ab.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_ab.log') if l.startswith('{')][-1]); print('$c', round(d['ms_per_step']*1000,1),'us')"
done; done
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "fast or cfg2" > gpurun_out/pt_ab.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt_ab.log
