for mode in 0 1; do for sh in "16 16 216" "18 18 218" "20 20 220" "22 22 222"; do set -- $sh; echo "LDU8W=$mode L4 $1x$2 $(LNORM_LDU8W=$mode python tools/one_search.py $1 $2 --d 4 --seed $3 --reps 4)"; done; done
timeout 1500 python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/r2b_pytest_gpu6.log 2>&1; tail -3 gpurun_out/r2b_pytest_gpu6.log
