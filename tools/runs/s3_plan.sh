python -m pytest tests/test_gpu_parity.py tests/test_gpu_exhaustive.py tests/test_gpu_batch.py tests/test_gpu_fullsize.py -q -m gpu -x --timeout 900 2>&1 | tail -2
for sh in "--n 24 --m 24 --d 2 --seed 4 --reps 20" "--n 24 --m 24 --d 1 --seed 4 --reps 20" "--n 26 --m 26 --d 1 --seed 5 --reps 10" "--n 28 --m 28 --d 2 --seed 5 --reps 10" "--n 22 --m 22 --d 2 --seed 3 --reps 20" "--n 30 --m 30 --d 1 --seed 5 --reps 5"; do echo "== $sh"; python tools/time_variants.py $sh; done
python tools/latency_probe.py
