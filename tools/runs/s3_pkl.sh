python tools/time_variants.py --n 36 --m 144 --d 1 --seed 136 --reps 3
python tools/time_variants.py --n 40 --m 160 --d 1 --seed 140 --reps 2
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x --timeout 900 -k "wide or 144 or 160 or 192 or hot_kernel" 2>&1 | tail -2
