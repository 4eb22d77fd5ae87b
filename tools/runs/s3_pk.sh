python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_exhaustive.py tests/test_gpu_batch.py -q -m gpu -x --timeout 900 2>&1 | tail -3
for sh in "--n 24 --m 24 --d 3 --seed 4" "--n 22 --m 22 --d 3 --seed 5" "--n 20 --m 20 --d 4 --seed 5" "--n 18 --m 18 --d 4 --seed 218" "--n 26 --m 24 --d 3 --seed 7"; do echo "== $sh"; python tools/time_variants.py $sh; done
