mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_wide3_gpu.py tests/test_fullsize_gpu.py tests/test_parity_gpu.py -x -q -k "wide3 or cfg3" > gpurun_out/pt_it7.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_it7.log
timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --profile --no-cpu-baseline > gpurun_out/bench_it7.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_it7.log') if l.startswith('{')][-1]); print('cfg3', round(d['ms_per_step']*1000,1),'us', json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))"
for gs in 1 0; do TTGPU_GRID_SORT=$gs timeout 600 python bench.py --config cfg5 --steps 20 --warmup 5 > gpurun_out/bench_cfg5_gs$gs.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_cfg5_gs$gs.log') if l.startswith('{')][-1]); print('cfg5 gridsort=$gs', d['ms_per_step'], d.get('sequential_ms_per_step'))"; done
