# f4 experiment: parity vs oracle, throughput vs the byte walk, ncu of the imma kernel; wide-row parity
timeout 300 python -m pytest tests/test_gpu_imma.py -q -x > gpurun_out/r2b_imma_pytest.log 2>&1; tail -15 gpurun_out/r2b_imma_pytest.log
timeout 300 python tools/bench_imma.py > gpurun_out/r2b_bench_imma.json 2>&1; cat gpurun_out/r2b_bench_imma.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:imma_l1_kernel -s 1 -c 1 -o gpurun_out/ncu_r2b_imma2 python tools/bench_imma.py --tiles-log2 18 --reps 1 --no-walk > gpurun_out/r2b_ncu_imma.log 2>&1; tail -3 gpurun_out/r2b_ncu_imma.log
