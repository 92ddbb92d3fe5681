# Round-2 closing pass: full GPU suite, smoke, every config's bench line, cfg2 launch list,
# per-kernel DRAM / FFMA counts, one ncu --set full of the five cfg2 kernels
TAG=${1:-r2f}
bash tools/gpu/final_r2.sh $TAG
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum --clock-control none -k regex:f3_ -c 40 --csv --log-file gpurun_out/kern_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_kernels.py gpurun_out/kern_$TAG.csv cfg2 gpurun_out/ncu_kernels_$TAG.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:f3_ -s 25 -c 5 -o gpurun_out/full_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncufull_$TAG.log 2>&1; echo "ncu full rc=$?"; tail -3 gpurun_out/ncufull_$TAG.log
