mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_cache_fast_gpu.py tests/test_cache_gpu.py -x -q > gpurun_out/pt_comb.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_comb.log
for i in 1 2; do for fc in 1 0; do for c in cfg2 cfg4 cfg2u; do
TTGPU_FUSE_COMB=$fc timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_comb.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_comb.log') if l.startswith('{')][-1]); print('fc=$fc $c', round(d['ms_per_step']*1000,1),'us')" || tail -3 gpurun_out/bench_comb.log
done; done; done
