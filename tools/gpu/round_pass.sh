#!/bin/bash
# One GPU pass: parity suite, smoke, bench, ncu launch list + per-kernel metrics, one ncu --set full.
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
lscpu > gpurun_out/lscpu_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_$TAG.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_$TAG.csv | tail -20
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum --clock-control none -k regex:f3_ -c 60 --csv --log-file gpurun_out/kern_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_kernels.py gpurun_out/kern_$TAG.csv cfg2 gpurun_out/ncu_kernels_$TAG.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:f3_ -s 45 -c 9 -o gpurun_out/full_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncufull_$TAG.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncufull_$TAG.log
