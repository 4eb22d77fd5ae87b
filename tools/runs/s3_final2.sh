# L_1 42x42 re-measure on the MERGE=0 build (s3_final ran a stale MRG=1 library), GPU suite again
python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/pytest_gpu_s3g.log 2>&1; tail -2 gpurun_out/pytest_gpu_s3g.log
c=l1_42x42
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8w?)_kernel" -c 1 -o /tmp/ncu_s3f_$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
NCU_BENCH_OUT=profiles/r02/walk_profiles.json python tools/ncu_bench.py $c /tmp/ncu_s3f_$c.ncu-rep > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ncu_s3f_$c.ncu-rep > gpurun_out/ncu_s3f_$c.json 2>/dev/null
sed -i "s/\"source\": \"ncu_s3f_$c.ncu-rep\"/\"source\": \"ncu_s3f_$c.ncu-rep (summary: ncu_s3f_$c.json)\"/" profiles/r02/walk_profiles.json
cp profiles/r02/walk_profiles.json gpurun_out/walk_profiles_s3f.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s3f_l1_42x42.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python bench.py > gpurun_out/bench_s3f_l1_42x42.json 2>/dev/null; tail -c 300 gpurun_out/bench_s3f_l1_42x42.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_s3f_torchrun1.json 2>/dev/null
python tools/sweep.py --budget-s 20 > gpurun_out/sweep_s3.jsonl 2>&1
python tools/latency_probe.py > gpurun_out/latency_s3.jsonl 2>&1
