mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_wide3_gpu.py tests/test_cache_fast_gpu.py -x -q > gpurun_out/pt_it3.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pt_it3.log
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_parity_gpu.py -x -q -k "cfg3" > gpurun_out/pt_it3_full.log 2>&1; echo "pytest full rc=$?"; tail -4 gpurun_out/pt_it3_full.log
timeout 300 python bench.py --config cfg3 --steps 5 --warmup 3 --profile --no-cpu-baseline > gpurun_out/bench_it3.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_it3.log') if l.startswith('{')][-1]); print(round(d['ms_per_step']*1000,1),'us', json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_w3_fwd|k_w3_bwd|k_head_fwd" -s 3 -c 3 -o gpurun_out/w3b_full python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_w3b.log 2>&1; echo "ncu rc=$?"
