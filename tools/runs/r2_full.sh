python -m pytest tests/ -q -m gpu -x --timeout 900 2>&1 | tail -4
compute-sanitizer --tool memcheck python tests/sanitize_cases.py > gpurun_out/r2_memcheck.txt 2>&1; tail -3 gpurun_out/r2_memcheck.txt
compute-sanitizer --tool racecheck python tests/sanitize_cases.py > gpurun_out/r2_racecheck.txt 2>&1; tail -3 gpurun_out/r2_racecheck.txt
for c in l3_24x24 l3_26x26 l4_18x18 marg_40x40 l2_24x24 l1_20x20; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_r2_$c.json 2>/dev/null; done
