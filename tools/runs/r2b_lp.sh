# lane pairs from 32 (128 columns) and 24 words (96 columns) vs one lane per unit; ncu of 34x136 vs 36x144
python tools/time_variants.py --n 38 --m 128 --seed 7 --reps 3 > gpurun_out/r2b_lp_38x128.jsonl 2>&1; cat gpurun_out/r2b_lp_38x128.jsonl
python tools/time_variants.py --n 32 --m 128 --seed 132 --reps 3 > gpurun_out/r2b_lp_32x128.jsonl 2>&1; cat gpurun_out/r2b_lp_32x128.jsonl
python tools/time_variants.py --n 36 --m 96 --seed 7 --reps 3 > gpurun_out/r2b_lp_36x96.jsonl 2>&1; cat gpurun_out/r2b_lp_36x96.jsonl
for s in "34 136 134" "36 144 136"; do set -- $s; timeout 600 ncu --set full --clock-control none -k regex:"walk_u8_kernel" -c 1 -o gpurun_out/ncu_r2b_l1_$1x$2 python tools/one_search.py $1 $2 --seed $3 > /dev/null 2>&1; done; ls gpurun_out/*.ncu-rep
