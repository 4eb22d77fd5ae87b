# full config-5 sweep on the per-family floor model (L_1 m = n and m = 4n, L_3 16..26)
timeout 2400 python tools/sweep.py --budget-s 20 > gpurun_out/r2b_sweep_full.jsonl 2>&1; cat gpurun_out/r2b_sweep_full.jsonl
