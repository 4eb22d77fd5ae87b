python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/pytest_gpu_s3h.log 2>&1; tail -2 gpurun_out/pytest_gpu_s3h.log
for c in l3_24x24 l3_26x26 l4_18x18; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8w?)(_pk)?_kernel" -c 1 -o /tmp/ncu_s3h_$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
  NCU_BENCH_OUT=profiles/r02/walk_profiles.json python tools/ncu_bench.py $c /tmp/ncu_s3h_$c.ncu-rep > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/ncu_s3h_$c.ncu-rep > gpurun_out/ncu_s3h_$c.json 2>/dev/null
  sed -i "s/\"source\": \"ncu_s3h_$c.ncu-rep\"/\"source\": \"ncu_s3h_$c.ncu-rep (summary: ncu_s3h_$c.json)\"/" profiles/r02/walk_profiles.json
done
cp profiles/r02/walk_profiles.json gpurun_out/walk_profiles_s3h.json
for c in l3_24x24 l3_26x26 l4_18x18; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3h_$c.json 2>/dev/null; done
python bench.py --config l2_24x24 --steps 3000 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3h_l2_24x24.json 2>/dev/null
python tools/sweep.py --l3-only --budget-s 20 > gpurun_out/sweep_s3h_l3.jsonl 2>&1
python tools/bench_next.py > gpurun_out/next_rows_s3h.jsonl 2>&1
