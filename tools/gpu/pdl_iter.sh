# PDL experiment: cfg2 bench with TTGPU_PDL=0/1/2 (+ fast-path parity under PDL)
mkdir -p gpurun_out
for m in 0 1 2; do
TTGPU_PDL=$m timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_pdl$m.log 2>&1; echo "pdl=$m rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_pdl$m.log').readline()); print(' ', round(d['ms_per_step']*1000,1),'us', 'e2e', round(d['e2e']['ms_per_step_median']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})" || tail -5 gpurun_out/bench_pdl$m.log
done
TTGPU_PDL=${1:-2} timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "fast_path or cfg2 or fused or deterministic" > gpurun_out/pt_pdl.log 2>&1; echo "pytest(PDL=${1:-2}) rc=$?"; tail -3 gpurun_out/pt_pdl.log
