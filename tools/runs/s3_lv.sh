for sh in "--n 24 --m 24 --d 3 --seed 4" "--n 22 --m 22 --d 4 --seed 5" "--n 26 --m 26 --d 3 --seed 226"; do echo "== $sh"; python tools/time_variants.py $sh; done
