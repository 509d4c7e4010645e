#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fp16 or int8_fused or fused_step or int8_kernels or pull_reducer" > gpurun_out/f_tests.log 2>&1
echo "rc $?" >> gpurun_out/f_tests.log
timeout 600 python bench.py > gpurun_out/bench_n1_int8.log 2>&1
timeout 300 python bench.py --method fp16 --no-cpu --no-e2e --steps 100 > gpurun_out/bench_n1_fp16.log 2>&1
timeout 300 python bench.py --method fp16 --no-cpu --no-e2e --steps 100 --no-step-fusion > gpurun_out/bench_n1_fp16_staged.log 2>&1
CMD="python scripts/profile_step.py --method int8 --steps 3"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_int8_ws" -s 1 -c 1 -o gpurun_out/int8_step $CMD > gpurun_out/ncu_int8.log 2>&1
CMD2="python scripts/profile_step.py --method qsgd --steps 3"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_int8_ws" -s 1 -c 1 -o gpurun_out/qsgd_step $CMD2 > gpurun_out/ncu_qsgd.log 2>&1
rm -f gpurun_out/config5_n1.jsonl
timeout 1200 python scripts/sweep.py --config 5 --out gpurun_out/config5_n1.jsonl > gpurun_out/sweep_c5_n1.log 2>&1
