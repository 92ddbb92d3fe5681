mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dlrm_gpu.py -x -q > gpurun_out/pt_dlrm.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pt_dlrm.log
timeout 600 python bench.py --config cfg5m --steps 10 --warmup 3 > gpurun_out/bench_cfg5m.log 2>&1; echo "cfg5m rc=$?"; tail -c 1500 gpurun_out/bench_cfg5m.log
for fs in 1 0; do TTGPU_FUSE_SB=$fs timeout 600 python bench.py --config cfg5 --steps 20 --warmup 5 > gpurun_out/bench_cfg5_fs$fs.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_cfg5_fs$fs.log') if l.startswith('{')][-1]); print('cfg5 fuse=$fs', d['ms_per_step'], d.get('sequential_ms_per_step'))"; done
