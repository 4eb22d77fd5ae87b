for c in l1_36x144; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8w?)(_pk)?_kernel" -c 1 -o /tmp/ncu_s3w_$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/ncu_s3w_$c.ncu-rep > gpurun_out/ncu_s3w_$c.json 2>/dev/null
  ncu -i /tmp/ncu_s3w_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_s3w_${c}_sass.csv 2>/dev/null
done
