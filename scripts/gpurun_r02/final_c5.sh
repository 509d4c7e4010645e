#!/bin/bash
# 2 GPUs: BASELINE config 5 on the final tree with the phase timers off during the timed steps —
# N = 1 (LOOPBACK, full grid 1 MiB .. 1 GiB) and N = 2 (4 MiB, 64 MiB, 1 GiB buckets).
mkdir -p gpurun_out/final_c5
O=gpurun_out/final_c5
python -m paper_2205_09470_b200.build > $O/build.log 2>&1
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29635"
timeout 1800 python scripts/sweep.py --config 5 --out $O/config5_n1.jsonl > $O/c5_n1.log 2>&1
timeout 1500 $T2 scripts/sweep.py --config 5 --sizes 20,24,28 --out $O/config5_n2.jsonl > $O/c5_n2.log 2>&1
