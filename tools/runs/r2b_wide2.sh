timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wide or hot_kernel" > gpurun_out/r2b_wide2_pytest.log 2>&1; tail -3 gpurun_out/r2b_wide2_pytest.log
timeout 1500 python tools/sweep.py --wide-only --budget-s 20 > gpurun_out/r2b_sweep_wide2.jsonl 2>&1; cut -c1-60,300-420 gpurun_out/r2b_sweep_wide2.jsonl
