for sh in "--n 14 --m 14 --d 4 --seed 5 --reps 20" "--n 15 --m 20 --d 4 --seed 6 --reps 20"; do echo "== $sh"; python tools/time_variants.py $sh; done
echo "== forced PR=3 (LNORM_LDU8W_PR=3) 18x18, 20x20"; LNORM_LDU8W_PR=3 python tools/time_variants.py --n 18 --m 18 --d 4 --seed 218 --reps 10; LNORM_LDU8W_PR=3 python tools/time_variants.py --n 20 --m 20 --d 4 --seed 5 --reps 5
echo "== product batch"; python tools/bench_next.py 2>&1 | grep '"L_4"' | cut -c1-300
echo "== nol4pr3 batch"; LNORM_LIB=paper_2503_21596_b200/_exp/liblnorm_nol4pr3.so python tools/bench_next.py 2>&1 | grep '"L_4"' | cut -c1-300
python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -q -m gpu -x --timeout 900 -k "L4 or ld or batch or packed" 2>&1 | tail -2
