mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_wide3_gpu.py tests/test_cache_fast_gpu.py tests/test_cache_gpu.py -x -q > gpurun_out/pt_it4.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pt_it4.log
for a in "--config cfg3"; do
timeout 300 python bench.py $a --steps 10 --warmup 5 --profile --no-cpu-baseline > gpurun_out/bench_it4.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_it4.log') if l.startswith('{')][-1]); print('$a', round(d['ms_per_step']*1000,1),'us', json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))" || tail -5 gpurun_out/bench_it4.log
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_w3_fwd|k_w3_bwd" -s 2 -c 2 -o gpurun_out/w3d_full python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_w3c.log 2>&1; echo "ncu rc=$?"
