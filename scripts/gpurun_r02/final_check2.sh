#!/bin/bash
# 2 GPUs: test_multigpu 2x1 / 1x2 through tests/dist_check.py (moved), config 1 latency (timers
# off) at N = 1 and 2, the sanitizer workload from tests/, a top-k bench line (roofline note).
mkdir -p gpurun_out/final_check2
O=gpurun_out/final_check2
python -m paper_2205_09470_b200.build > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q -rA > $O/test_multigpu_n2.log 2>&1; echo "rc $?" >> $O/test_multigpu_n2.log
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29634"
timeout 600 python scripts/sweep.py --config 1 --out $O/config1_n1.jsonl > $O/c1_n1.log 2>&1
timeout 600 $T2 scripts/sweep.py --config 1 --out $O/config1_n2.jsonl > $O/c1_n2.log 2>&1
timeout 600 python tests/sanitize_workload.py > $O/sanitize_workload.log 2>&1; echo "rc $?" >> $O/sanitize_workload.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 30 --method topk > $O/bench_topk1.json 2> $O/bench_topk1.err
