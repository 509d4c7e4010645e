#!/bin/bash
# 1 GPU: top-k tie-pass early exit (parity), and the pipelined step's stage-pass grid (CTAs per
# SM) x staggered halves, at rho = 1 % and 10 %.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "topk" > gpurun_out/o_tests.log 2>&1
echo "tests rc $?" >> gpurun_out/o_tests.log
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 30"
for D in 0.01 0.1; do
  for X in 0 1; do
    for C in 0 1; do
      NEBULA_EXPERIMENT_STAGGER=$X NEBULA_EXPERIMENT_STAGE_CTAS=$C $B --method topk --density $D > gpurun_out/o_topk_${D}_s${X}_c${C}.log 2>&1
    done
  done
  $B --method topk --density $D --no-pipeline > gpurun_out/o_topk_${D}_nopipe.log 2>&1
done
