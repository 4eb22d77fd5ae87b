python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/pytest_gpu_s3v.log 2>&1; tail -2 gpurun_out/pytest_gpu_s3v.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_s3v.log 2>&1; tail -1 gpurun_out/smoke_s3v.log
python bench.py > gpurun_out/bench_s3v_default.json 2>/dev/null; tail -c 250 gpurun_out/bench_s3v_default.json
python bench.py --config l3_24x24 --steps 300 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3v_l3_24x24.json 2>/dev/null; tail -c 150 gpurun_out/bench_s3v_l3_24x24.json
