#!/bin/bash
# 1 GPU: the fused step's A->B lead (1 / 2 / 3 buckets), top-k after skipping the wide-resolve
# launches, and the serialized top-k launch list at rho = 1 % (per-kernel durations).
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "topk" > gpurun_out/n_tests.log 2>&1
echo "tests rc $?" >> gpurun_out/n_tests.log
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 30"
for L in 1 2 3; do
  NEBULA_EXPERIMENT_LEAD=$L $B --method int8 > gpurun_out/n_int8_lead$L.log 2>&1
done
NEBULA_EXPERIMENT_LEAD=1 $B --method fp8 > gpurun_out/n_fp8_lead1.log 2>&1
$B --method fp8 > gpurun_out/n_fp8_lead2.log 2>&1
$B --method topk > gpurun_out/n_topk1.log 2>&1
$B --method topk --density 0.1 > gpurun_out/n_topk10.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n_topk1_launches.csv \
  python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 --method topk --no-pipeline > gpurun_out/n_ncu.log 2>&1
