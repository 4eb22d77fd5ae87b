for sh in "24 24 4 3" "26 26 226 3" "20 20 220 4" "22 22 222 4"; do set -- $sh; echo "L$4 $1x$2 $(python tools/one_search.py $1 $2 --d $4 --seed $3 --reps 4)"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8w?)_kernel" -c 1 -o /tmp/ncu_r2f_l3_24x24 python bench.py --config l3_24x24 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ncu_r2f_l3_24x24.ncu-rep > gpurun_out/ncu_r2f_l3_24x24.json 2>/dev/null
cp profiles/r02/walk_profiles.json gpurun_out/walk_profiles_l3.json; NCU_BENCH_OUT=gpurun_out/walk_profiles_l3.json python tools/ncu_bench.py l3_24x24 /tmp/ncu_r2f_l3_24x24.ncu-rep
timeout 900 python -m pytest tests/ -q -m gpu -x -k "3 or ld or L3 or L4 or batch or exhaustive" > gpurun_out/r2b_l3b_pytest.log 2>&1; tail -2 gpurun_out/r2b_l3b_pytest.log
