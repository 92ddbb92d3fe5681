mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "fast or cfg2 or fused" > gpurun_out/pt_sr.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt_sr.log
for i in 1 2; do for v in 0 1 2 3; do
TTGPU_SROWS_CTAS_PER_SM=$v timeout 300 python bench.py --config cfg2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sr.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_sr.log') if l.startswith('{')][-1]); print('srows/sm=$v cfg2', round(d['ms_per_step']*1000,1),'us')"
done; done
