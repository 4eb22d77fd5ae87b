# session-3 measurement pass: GPU suite, sanitizers, smoke, ncu of the bench launches, launch list, bench lines
python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/pytest_gpu_s3f.log 2>&1; tail -2 gpurun_out/pytest_gpu_s3f.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_s3f.log 2>&1; tail -1 gpurun_out/smoke_s3f.log
compute-sanitizer --tool memcheck python tests/sanitize_cases.py > gpurun_out/compute_sanitizer_memcheck_s3.txt 2>&1; tail -2 gpurun_out/compute_sanitizer_memcheck_s3.txt
compute-sanitizer --tool racecheck python tests/sanitize_cases.py > gpurun_out/compute_sanitizer_racecheck_s3.txt 2>&1; tail -2 gpurun_out/compute_sanitizer_racecheck_s3.txt
for c in l1_42x42 marg_40x40 l3_24x24 l4_18x18 l2_24x24 l3_26x26; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8w?)_kernel" -c 1 -o /tmp/ncu_s3f_$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
  NCU_BENCH_OUT=profiles/r02/walk_profiles.json python tools/ncu_bench.py $c /tmp/ncu_s3f_$c.ncu-rep > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/ncu_s3f_$c.ncu-rep > gpurun_out/ncu_s3f_$c.json 2>/dev/null
  sed -i "s/\"source\": \"ncu_s3f_$c.ncu-rep\"/\"source\": \"ncu_s3f_$c.ncu-rep (summary: ncu_s3f_$c.json)\"/" profiles/r02/walk_profiles.json
done
cp profiles/r02/walk_profiles.json gpurun_out/walk_profiles_s3f.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s3f_l1_42x42.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python bench.py > gpurun_out/bench_s3f_l1_42x42.json 2>/dev/null; tail -c 300 gpurun_out/bench_s3f_l1_42x42.json
for c in marg_40x40 l3_24x24 l3_26x26 l4_18x18 l1_36x144 l1_40x160; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3f_$c.json 2>/dev/null; done
for c in l2_24x24 l1_20x20; do python bench.py --config $c --steps 3000 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3f_$c.json 2>/dev/null; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_s3f_reference.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_s3f_torchrun1.json 2>/dev/null
ls gpurun_out
