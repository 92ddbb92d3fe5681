mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/pt_c3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_c3.log
timeout 400 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg3.log').readline()); print(d['value'], d['ms_per_step'], d['phases_ms'])"
timeout 300 python bench.py --fast-forward --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ffma.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_ffma.log').readline()); print('ffma', d['value'], d['ms_per_step'], d['phases_ms'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_chunk_reduce|k_tail_pool|k_head_bwd" -s 3 -c 4 -o gpurun_out/c3 python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
