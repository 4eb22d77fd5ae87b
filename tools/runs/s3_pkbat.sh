python -m pytest tests/test_gpu_batch.py tests/test_gpu_exhaustive.py tests/test_gpu_boundary.py -q -m gpu -x --timeout 900 2>&1 | tail -2
python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 900 -k "packed_walk_sliced" 2>&1 | tail -2
echo "== product"; python tools/bench_next.py 2>&1 | grep -v '"L_1"\|"L_marg"\|"L_2"' | cut -c1-330
echo "== nopkbat"; LNORM_LIB=paper_2503_21596_b200/_exp/liblnorm_nopkbat.so python tools/bench_next.py 2>&1 | grep -v '"L_1"\|"L_marg"\|"L_2"' | cut -c1-330
