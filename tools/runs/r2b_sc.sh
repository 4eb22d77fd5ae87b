timeout 900 python -m pytest tests/test_gpu_selfcheck.py -q -x > gpurun_out/r2b_sc_pytest.log 2>&1; tail -15 gpurun_out/r2b_sc_pytest.log
