# d-ary small-search cost model + device-side batch guard stats: GPU suite, L_3 sweep rows, batch numbers, L_4 bench
timeout 1500 python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/r2b_pytest_gpu4.log 2>&1; tail -3 gpurun_out/r2b_pytest_gpu4.log
timeout 900 python tools/bench_next.py --batch-only > gpurun_out/r2b_next_batch3.jsonl 2>&1; cat gpurun_out/r2b_next_batch3.jsonl | cut -c1-260
timeout 900 python tools/sweep.py --budget-s 20 > gpurun_out/r2b_sweep_full2.jsonl 2>&1; grep "L_3" gpurun_out/r2b_sweep_full2.jsonl | cut -c1-330
for c in l4_18x18 l3_24x24; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_$c.json 2>/dev/null; cut -c1-200 gpurun_out/r2b_bench_$c.json; done
