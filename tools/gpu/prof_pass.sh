#!/bin/bash
# Round profile pass: FP32 peak, bench, ncu launch metrics, ncu --set full of every fast-path kernel
TAG=$1
mkdir -p gpurun_out
./tools/ffma_peak > gpurun_out/fp32_peak.json; cat gpurun_out/fp32_peak.json
mkdir -p profiles; cp gpurun_out/fp32_peak.json profiles/fp32_peak.json
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench$TAG.log 2>&1; echo "bench rc=$?"; tail -c 4000 gpurun_out/bench$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum --clock-control none -c 60 --csv --log-file gpurun_out/kern$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_kernels.py gpurun_out/kern$TAG.csv cfg2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:f3_ -s 40 -c 8 -o gpurun_out/full$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncufull$TAG.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncufull$TAG.log
