python tools/time_variants.py --n 42 --m 42 --d 1 --seed 2 --reps 2
python tools/time_variants.py --n 32 --m 128 --d 1 --seed 1 --reps 3
python tools/time_variants.py --n 20 --m 20 --d 1 --seed 1 --reps 5
for c in l3_24x24 l1_42x42; do
  ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8w?)_kernel" -c 1 -o gpurun_out/ncu_s3_$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_s3_$c.log 2>&1; tail -2 gpurun_out/ncu_s3_$c.log
done
