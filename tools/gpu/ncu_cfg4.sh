mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sanitizer_gpu.py -x -q > gpurun_out/pt_san.log 2>&1; echo "sanitizer rc=$?"; tail -3 gpurun_out/pt_san.log
timeout 300 python bench.py --config cfg4 --steps 20 --warmup 5 --profile --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_c4.log') if l.startswith('{')][-1]); print(round(d['ms_per_step']*1000,1),'us', json.dumps({k:round(v*1000,1) for k,v in d.get('phases_ms',{}).items()}))"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"f3_gsort|f3_srows|k_slot" -s 12 -c 4 -o gpurun_out/cfg4_full python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"f3_gsort" -s 6 -c 1 -o gpurun_out/cfg2z_gsort python bench.py --config cfg2z12 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c2z.log 2>&1; echo "ncu rc=$?"
