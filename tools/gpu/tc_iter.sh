# tcgen05 head-backward iteration: cfg3 parity, cfg3 bench with and without the tensor path,
# optional ncu --set full of both head kernels (arg "ncu")
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q -k "cfg3 or tensor" > gpurun_out/pt_tc.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pt_tc.log
for f in "" "--ffma-backward"; do
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline $f > gpurun_out/bench_cfg3$f.log 2>&1; echo "bench $f rc=$?"
python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_cfg3$f.log').readline()); print(d['value'], d['ms_per_step'], json.dumps({k:round(v,3) for k,v in d['phases_ms'].items()}))" || tail -5 gpurun_out/bench_cfg3$f.log
done
if [ "$1" = "ncu" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_head_bwd -c 1 -o gpurun_out/head_tc python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_head_tc.log 2>&1; echo "ncu tc rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_head_bwd -c 1 -o gpurun_out/head_ffma python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline --ffma-backward > gpurun_out/ncu_head_ffma.log 2>&1; echo "ncu ffma rc=$?"
fi
