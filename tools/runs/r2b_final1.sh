# ncu captures of the exact bench launches, summarised ON the box (reports are large), plus the launch list
cp profiles/r02/walk_profiles.json gpurun_out/walk_profiles_r2f.json
for c in l1_42x42 marg_40x40 l3_24x24 l4_18x18 l2_24x24 l3_26x26; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8w?)_kernel" -c 1 -o /tmp/ncu_r2f_$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
  NCU_BENCH_OUT=gpurun_out/walk_profiles_r2f.json python tools/ncu_bench.py $c /tmp/ncu_r2f_$c.ncu-rep > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/ncu_r2f_$c.ncu-rep > gpurun_out/ncu_r2f_$c.json 2>/dev/null
  sed -i "s/\"source\": \"ncu_r2f_$c.ncu-rep\"/\"source\": \"ncu_r2f_$c.ncu-rep (summary: ncu_r2f_$c.json)\"/" gpurun_out/walk_profiles_r2f.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2f_l1_42x42.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/
