#!/bin/bash
# 4 GPUs: BASELINE config 5 at N = 4 on the final tree, phase timers off during the timed steps.
mkdir -p gpurun_out/final_c5
O=gpurun_out/final_c5
python -m paper_2205_09470_b200.build > $O/build4.log 2>&1
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29637"
timeout 2000 $T4 scripts/sweep.py --config 5 --sizes 20,24,28 --out $O/config5_n4.jsonl > $O/c5_n4.log 2>&1
