# ncu --set full of the cfg3 wide-row kernels (one launch each) + cache/wide3 tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cache_fast_gpu.py tests/test_wide3_gpu.py -x -q > gpurun_out/pt_w3.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pt_w3.log
timeout 300 python bench.py --config cfg3 --steps 5 --warmup 3 --profile --no-cpu-baseline > gpurun_out/bench_w3.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_w3.log') if l.startswith('{')][-1]); print(round(d['ms_per_step']*1000,1),'us', json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_w3|k_head_fwd|k_pool_rows|k_head_g0" -s 8 -c 6 -o gpurun_out/w3_full python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_w3.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_w3.log
