#!/bin/bash
# 2 GPUs: the size-aware P = 2 policy (FP16 / QSGD pull only on >= 8 MiB buckets).
mkdir -p gpurun_out/final_check3
O=gpurun_out/final_check3
python -m paper_2205_09470_b200.build > $O/build.log 2>&1
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29636"
timeout 600 $T2 scripts/sweep.py --config 1 --out $O/config1_n2.jsonl > $O/c1_n2.log 2>&1
timeout 600 $T2 bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e --method fp16 > $O/bench_n2_fp16.log 2>&1
timeout 600 $T2 bench.py --gpus 2 --steps 50 --warmup 5 > $O/bench_n2_int8.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -q -rA -k "2-1" > $O/test_multigpu_2x1.log 2>&1; echo "rc $?" >> $O/test_multigpu_2x1.log
