# round 2 (session 2) first box call: GPU suite, headline bench, wide-row bench + ncu of its walk launch
python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/r2b_pytest_gpu.log 2>&1; tail -4 gpurun_out/r2b_pytest_gpu.log
python bench.py > gpurun_out/r2b_bench_default.json 2> gpurun_out/r2b_bench_default.err; cat gpurun_out/r2b_bench_default.json
for c in l1_36x144 l1_40x160; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_$c.json 2>/dev/null; cat gpurun_out/r2b_bench_$c.json; done
ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8)_kernel" -c 1 -o gpurun_out/ncu_r2b_l1_36x144 python bench.py --config l1_36x144 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
