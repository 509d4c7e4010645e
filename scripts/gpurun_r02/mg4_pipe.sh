#!/bin/bash
# 4 GPUs: the two-stream pipelined step at G > 1 (P2P intra hop) — parity (2x2, 1x4) and the
# BASELINE config 3 adapter bench with and without the pipeline.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q -rA -k "4-2 or 4-4" > gpurun_out/test_multigpu_n4_pipe.log 2>&1
echo "multigpu rc $?" >> gpurun_out/test_multigpu_n4_pipe.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631"
B="timeout 600 $TR bench.py --gpus 4 --steps 50 --warmup 5 --no-e2e --workload ernie-m-large-adapters"
for G in 2 4; do
  for M in int8 topk fp16; do
    $B --gpus-per-cluster $G --method $M > gpurun_out/bench_pipe_${G}_${M}.log 2>&1
    $B --gpus-per-cluster $G --method $M --no-pipeline > gpurun_out/bench_nopipe_${G}_${M}.log 2>&1
  done
done
