python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x --timeout 900 2>&1 | tail -2
for sh in "--n 24 --m 24 --d 3 --seed 4" "--n 26 --m 26 --d 3 --seed 226" "--n 20 --m 20 --d 4 --seed 5" "--n 22 --m 22 --d 4 --seed 5" "--n 22 --m 28 --d 3 --seed 9"; do echo "== $sh"; python tools/time_variants.py $sh; done
