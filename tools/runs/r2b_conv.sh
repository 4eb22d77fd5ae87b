# L_3 all-H: max-plus subset convolution (product) vs the 81-candidate form (conv0); envelope; ncu of the new L_3 walk
python tools/time_variants.py --n 24 --m 24 --d 3 --seed 4 --reps 5 > gpurun_out/r2b_conv_24.jsonl 2>&1; cat gpurun_out/r2b_conv_24.jsonl
python tools/time_variants.py --n 26 --m 26 --d 3 --seed 226 --reps 3 > gpurun_out/r2b_conv_26.jsonl 2>&1; cat gpurun_out/r2b_conv_26.jsonl
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "L3 or ld or d3" > gpurun_out/r2b_conv_pytest.log 2>&1; tail -2 gpurun_out/r2b_conv_pytest.log
timeout 600 python tools/envelope.py > gpurun_out/r2b_envelope.jsonl 2>&1; cat gpurun_out/r2b_envelope.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"walk_(u8|ldu8w?)_kernel" -c 1 -o gpurun_out/ncu_r2b_l3_24x24 python bench.py --config l3_24x24 --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1; ls gpurun_out/*.ncu-rep
