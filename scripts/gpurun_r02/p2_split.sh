#!/bin/bash
# 2 GPUs: the fused INT8 step over P2P pull at P = 2 with every pull warp split (configs 4..10).
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632"
B2="timeout 600 $T2 bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e --no-cpu --exchange pull"
for C in 4 5 6 7 8 9 10; do $B2 --step-config $C > gpurun_out/p2split_$C.log 2>&1; done
$B2 --method qsgd --step-config 1 > gpurun_out/p2split_qsgd_1.log 2>&1
