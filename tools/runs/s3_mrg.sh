python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "merged or sampled or planted or full" 2>&1 | tail -3
python tools/time_variants.py --n 42 --m 42 --d 1 --seed 2 --reps 2
python tools/time_variants.py --n 36 --m 38 --d 1 --seed 2 --reps 2
