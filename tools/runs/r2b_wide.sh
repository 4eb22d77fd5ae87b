# wide-row A/B: even word counts (36/42 words) vs round-1 rounding to 8 (40/48), register bound of the lane-pair instance
python tools/time_variants.py --n 36 --m 144 --seed 136 --reps 3 > gpurun_out/r2b_wide_36x144.jsonl 2>&1
python tools/time_variants.py --n 40 --m 160 --seed 140 --reps 2 > gpurun_out/r2b_wide_40x160.jsonl 2>&1
cat gpurun_out/r2b_wide_*.jsonl
