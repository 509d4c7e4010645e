#!/bin/bash
# 1 GPU: no-EF ring-A tiles (INT8 fused step without EF), the register zero-store sparse
# reducer, the staggered two-half top-k step: parity + bench.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "topk or int8 or pull_reducer or e5m2 or qsgd or fp8" > gpurun_out/m_tests.log 2>&1
echo "tests rc $?" >> gpurun_out/m_tests.log
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 30"
$B --method int8 --no-ef > gpurun_out/m_int8_noef.log 2>&1
$B --method int8 > gpurun_out/m_int8.log 2>&1
$B --method qsgd --no-ef > gpurun_out/m_qsgd_noef.log 2>&1
for D in 0.01 0.1; do
  $B --method topk --density $D > gpurun_out/m_topk_${D}.log 2>&1
  $B --method topk --density $D --no-pipeline > gpurun_out/m_topk_${D}_nopipe.log 2>&1
done
