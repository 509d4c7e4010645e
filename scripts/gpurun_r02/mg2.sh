#!/bin/bash
# 2-GPU pass: multi-process parity over NCCL/IPC (test_multigpu: 2x1, 1x2), bench at N = 2
# (P = 2 and the 1 x 2 hierarchical adapters config), config 1 at N = 2.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q -rA > gpurun_out/test_multigpu_n2.log 2>&1
echo "multigpu rc $?" >> gpurun_out/test_multigpu_n2.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
timeout 600 $TR bench.py --gpus 2 --steps 50 --warmup 5 > gpurun_out/bench_n2_int8.log 2>&1
timeout 600 $TR bench.py --gpus 2 --steps 50 --warmup 5 --gpus-per-cluster 2 --workload ernie-m-large-adapters --no-e2e > gpurun_out/bench_n2_1x2_adapters.log 2>&1
timeout 600 $TR bench.py --gpus 2 --steps 50 --warmup 5 --gpus-per-cluster 2 --workload ernie-m-large-adapters --no-e2e --method topk > gpurun_out/bench_n2_1x2_adapters_topk.log 2>&1
rm -f gpurun_out/config1_n2.jsonl
timeout 600 $TR scripts/sweep.py --config 1 --out gpurun_out/config1_n2.jsonl > gpurun_out/sweep_c1_n2.log 2>&1
