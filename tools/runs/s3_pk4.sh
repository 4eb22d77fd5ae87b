for sh in "--n 16 --m 16 --d 3 --seed 216 --reps 20" "--n 18 --m 18 --d 3 --seed 218 --reps 20" "--n 19 --m 24 --d 3 --seed 3 --reps 10"; do echo "== $sh"; python tools/time_variants.py $sh; done
echo "== forced PR=4, 22x22 and 24x24"; LNORM_LDU8W_PR=4 python tools/time_variants.py --n 22 --m 22 --d 3 --seed 5; LNORM_LDU8W_PR=4 python tools/time_variants.py --n 24 --m 24 --d 3 --seed 4
LNORM_LIB=paper_2503_21596_b200/_exp/liblnorm_pk4.so python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "paired_rows_every or allh or packed or l3_l4 or ld_workload" 2>&1 | tail -2
for c in l3_24x24 l4_18x18; do python bench.py --config $c --steps 300 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3z_$c.json 2>/dev/null; tail -c 150 gpurun_out/bench_s3z_$c.json; done
