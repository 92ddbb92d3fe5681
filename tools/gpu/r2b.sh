timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2b_pytest.log 2>&1; echo pytest=$? >> gpurun_out/r2b_pytest.log
tail -5 gpurun_out/r2b_pytest.log
