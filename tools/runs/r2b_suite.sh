timeout 1500 python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/r2b_pytest_gpu5.log 2>&1; tail -3 gpurun_out/r2b_pytest_gpu5.log
