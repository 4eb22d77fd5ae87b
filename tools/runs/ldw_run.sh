python -m pytest tests/test_gpu_parity.py -q -x -k "ldu8 or ld_workload or l3_l4 or hot_kernel or ties" 2>&1 | tail -2
python -m pytest tests/test_gpu_fullsize.py -q -x -k "L3" 2>&1 | tail -2
python -m pytest tests/test_gpu_exhaustive.py -q -x -k "L3" 2>&1 | tail -2
for sh in "24 24 4" "26 26 226" "24 40 5" "20 20 220"; do set -- $sh
python tools/ab_env.py --n $1 --m $2 --d 3 --seed $3 --env "" ; done
ncu --set full --clock-control none --import-source on -k regex:"walk_ldu8w_kernel" -c 1 -o gpurun_out/ncu_r2_l3_24x24_w4e python bench.py --config l3_24x24 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
