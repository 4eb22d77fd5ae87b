for sm in 10 11 12 13; do for sh in "34 136 134" "36 144 136" "32 128 132"; do set -- $sh; echo "smin=$sm $1x$2 $(LNORM_U8_SMIN=$sm python tools/one_search.py $1 $2 --seed $3 --reps 4)"; done; done
