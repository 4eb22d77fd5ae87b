python bench.py --config l4_22x22 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3z_l4_22x22.json 2>/dev/null; tail -c 300 gpurun_out/bench_s3z_l4_22x22.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8w?)(_pk)?_kernel" -c 1 -o /tmp/ncu_s3z_l4_22x22 python bench.py --config l4_22x22 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
NCU_BENCH_OUT=profiles/r02/walk_profiles.json python tools/ncu_bench.py l4_22x22 /tmp/ncu_s3z_l4_22x22.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ncu_s3z_l4_22x22.ncu-rep > gpurun_out/ncu_s3z_l4_22x22.json 2>/dev/null
sed -i "s/\"source\": \"ncu_s3z_l4_22x22.ncu-rep\"/\"source\": \"ncu_s3z_l4_22x22.ncu-rep (summary: ncu_s3z_l4_22x22.json)\"/" profiles/r02/walk_profiles.json
cp profiles/r02/walk_profiles.json gpurun_out/walk_profiles_s3z.json
python bench.py --config l4_22x22 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3z_l4_22x22.json 2>/dev/null
python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/pytest_gpu_s3y.log 2>&1; tail -2 gpurun_out/pytest_gpu_s3y.log
