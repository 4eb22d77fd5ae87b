for pr in 4 5; do for sh in "24 24 4" "26 26 226" "22 22 222" "20 20 220"; do set -- $sh; echo "PR<=$pr $1x$2 $(LNORM_LDU8W_PR=$pr python tools/one_search.py $1 $2 --d 3 --seed $3 --reps 4)"; done; done
timeout 900 python -m pytest tests/ -q -m gpu -x -k "3 or ld or L3 or batch or exhaustive" > gpurun_out/r2b_pr5_pytest.log 2>&1; tail -3 gpurun_out/r2b_pr5_pytest.log
