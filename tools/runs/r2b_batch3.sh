# batched byte kernels after the stride-alignment fix: batch tests, whole GPU suite, sanitizers
timeout 600 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/r2b_batch_pytest.log 2>&1; tail -3 gpurun_out/r2b_batch_pytest.log
timeout 1500 python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/r2b_pytest_gpu3.log 2>&1; tail -3 gpurun_out/r2b_pytest_gpu3.log
timeout 900 compute-sanitizer --tool memcheck python tests/sanitize_cases.py > gpurun_out/r2b_memcheck.txt 2>&1; tail -3 gpurun_out/r2b_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck python tests/sanitize_cases.py > gpurun_out/r2b_racecheck.txt 2>&1; tail -3 gpurun_out/r2b_racecheck.txt
