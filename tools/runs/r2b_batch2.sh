# batched byte kernels: parity, the whole GPU suite, batch-regime numbers, headline bench
timeout 600 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/r2b_batch_pytest.log 2>&1; tail -15 gpurun_out/r2b_batch_pytest.log
timeout 1200 python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/r2b_pytest_gpu2.log 2>&1; tail -4 gpurun_out/r2b_pytest_gpu2.log
timeout 900 python tools/bench_next.py --batch-only > gpurun_out/r2b_next_batch2.jsonl 2>&1; cat gpurun_out/r2b_next_batch2.jsonl
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b_bench2.json 2>/dev/null; cut -c1-300 gpurun_out/r2b_bench2.json
