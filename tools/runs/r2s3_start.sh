set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/pytest_gpu_s3.log 2>&1; tail -4 gpurun_out/pytest_gpu_s3.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_s3.log 2>&1; tail -2 gpurun_out/smoke_s3.log
python bench.py > gpurun_out/bench_s3_default.json 2> gpurun_out/bench_s3_default.err; cat gpurun_out/bench_s3_default.json
