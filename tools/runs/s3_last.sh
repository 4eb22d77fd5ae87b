# final pass on the final build: GPU suite, smoke, every bench line, reference arm, torchrun, launch list
python -m pytest tests/ -q -m gpu -x --timeout 900 > gpurun_out/pytest_gpu_s3z.log 2>&1; tail -2 gpurun_out/pytest_gpu_s3z.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_s3z.log 2>&1; tail -1 gpurun_out/smoke_s3z.log
python bench.py > gpurun_out/bench_s3z_l1_42x42.json 2>/dev/null; tail -c 200 gpurun_out/bench_s3z_l1_42x42.json
for c in marg_40x40 l3_24x24 l3_26x26 l4_18x18 l1_36x144 l1_40x160; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3z_$c.json 2>/dev/null; done
for c in l2_24x24 l1_20x20; do python bench.py --config $c --steps 3000 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s3z_$c.json 2>/dev/null; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_s3z_reference.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_s3z_torchrun1.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_s3z_l3_24x24.csv python bench.py --config l3_24x24 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | wc -l
