# Fast-path iteration on the GPU box: the parity suite, cfg2 and cfg2u bench lines (phase times), ncu launch list.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pt_iter.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pt_iter.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_iter.log').readline()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e'].get('pcie_best_GBs'), d['e2e']['ms_per_step_median'], d['phases_ms'])" || tail -5 gpurun_out/bench_iter.log
timeout 300 python bench.py --config cfg2u --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/bench_iter_u.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_iter_u.log').readline()); print('cfg2u', d['value'], d['ms_per_step'], d['phases_ms'])" || tail -5 gpurun_out/bench_iter_u.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:f3_ -c 40 --csv --log-file gpurun_out/launches_iter.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_iter.csv | tail -12
