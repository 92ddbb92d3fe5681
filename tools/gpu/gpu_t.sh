mkdir -p gpurun_out
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe2.log 2>&1; echo "probe rc=$?"; tail -40 gpurun_out/e2e_probe2.log
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k data_parallel > gpurun_out/dp.log 2>&1; echo "dp rc=$?"; tail -15 gpurun_out/dp.log
