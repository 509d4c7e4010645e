#!/bin/bash
# 2 GPUs: P = 2 exchange policy — staged push (auto) vs the fused step over P2P pull, per codec.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631"
B="timeout 600 $TR bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e"
for M in int8 fp16 topk fp8 qsgd; do
  $B --method $M > gpurun_out/p2_${M}_auto.log 2>&1
  $B --method $M --exchange pull > gpurun_out/p2_${M}_pull.log 2>&1
done
$B --method int8 --exchange nccl > gpurun_out/p2_int8_nccl.log 2>&1
