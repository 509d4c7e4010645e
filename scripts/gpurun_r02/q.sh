#!/bin/bash
# 1 GPU: the multi-CTA resolve threshold (candidates per bucket above which the resolve is
# spread over the whole GPU): parity at a low threshold, bench at 131072 / 32768 / 8192.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
NEBULA_EXPERIMENT_WIDE_MIN=8192 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "topk" > gpurun_out/q_tests.log 2>&1
echo "tests rc $?" >> gpurun_out/q_tests.log
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 30"
for D in 0.01 0.1; do
  for W in 131072 32768 8192; do
    NEBULA_EXPERIMENT_WIDE_MIN=$W $B --method topk --density $D > gpurun_out/q_topk_${D}_w${W}.log 2>&1
  done
  NEBULA_EXPERIMENT_WIDE_MIN=32768 $B --method topk --density $D --no-pipeline > gpurun_out/q_topk_${D}_w32768_nopipe.log 2>&1
done
