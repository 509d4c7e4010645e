#!/bin/bash
# 2 GPUs: BASELINE config 1 on the final tree (N = 1 LOOPBACK and N = 2 over NVLink), config 5
# at N = 1 (full grid) and N = 2 (2^24 / 2^28 buckets), ncu of the SFU-free QSGD fused step.
mkdir -p gpurun_out/final_sweeps
O=gpurun_out/final_sweeps
python -m paper_2205_09470_b200.build > $O/build.log 2>&1
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633"
timeout 600 python scripts/sweep.py --config 1 --out $O/config1_n1.jsonl > $O/c1_n1.log 2>&1
timeout 600 $T2 scripts/sweep.py --config 1 --out $O/config1_n2.jsonl > $O/c1_n2.log 2>&1
timeout 1500 python scripts/sweep.py --config 5 --out $O/config5_n1.jsonl > $O/c5_n1.log 2>&1
timeout 1200 $T2 scripts/sweep.py --config 5 --sizes 24,28 --out $O/config5_n2.jsonl > $O/c5_n2.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --clock-control none -k regex:k_int8_ws -s 2 -c 1 --csv --page raw \
  python scripts/profile_step.py --method qsgd --steps 3 > $O/ncu_qsgd_raw.csv 2> $O/ncu_qsgd.err
