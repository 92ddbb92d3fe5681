mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q -k "cfg3 or tensor" > gpurun_out/pt_tc.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_tc.log
for f in "" "--ffma-backward"; do
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline $f > gpurun_out/bench_cfg3$f.log 2>&1; echo "bench $f rc=$?"
python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_cfg3$f.log').readline()); print(d['value'], d['ms_per_step'], json.dumps({k:round(v,3) for k,v in d['phases_ms'].items()}))" || tail -5 gpurun_out/bench_cfg3$f.log
done
