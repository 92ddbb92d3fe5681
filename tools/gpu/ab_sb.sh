mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_cache_fast_gpu.py tests/test_wide3_gpu.py -x -q > gpurun_out/pt_sb.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_sb.log
for i in 1 2; do for fs in 1 0; do for c in cfg2 cfg4; do
TTGPU_FUSE_SB=$fs timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sb.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_sb.log') if l.startswith('{')][-1]); print('fuse=$fs $c', round(d['ms_per_step']*1000,1),'us')" || tail -3 gpurun_out/bench_sb.log
done; done; done
timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --profile --no-cpu-baseline > gpurun_out/bench_sb3.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_sb3.log') if l.startswith('{')][-1]); print('cfg3', round(d['ms_per_step']*1000,1),'us', json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))"
