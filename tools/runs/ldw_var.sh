python tools/time_variants.py --n 24 --m 24 --d 3 --seed 4 --reps 3
