# batch-regime breakdown (walk vs total) and the m = 4n wide-row sweep on the per-family floor model
timeout 900 python tools/bench_next.py --batch-only > gpurun_out/r2b_next_batch.jsonl 2>&1; cat gpurun_out/r2b_next_batch.jsonl
timeout 1500 python tools/sweep.py --wide-only --budget-s 20 > gpurun_out/r2b_sweep_wide.jsonl 2>&1; cat gpurun_out/r2b_sweep_wide.jsonl
timeout 300 python tools/latency_probe.py > gpurun_out/r2b_lat.jsonl 2>&1; tail -20 gpurun_out/r2b_lat.jsonl
