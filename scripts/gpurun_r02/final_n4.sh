#!/bin/bash
# Final 4-GPU pass of round 2: multi-process parity (2x1, 1x2, 4x1, 2x2, 1x4), bench lines at
# N = 2 and 4 on the final tree (exchange auto policy), hierarchical adapters, reference arm.
mkdir -p gpurun_out/final_n4
O=gpurun_out/final_n4
python -m paper_2205_09470_b200.build > $O/build.log 2>&1
timeout 2700 python -m pytest tests/test_multigpu.py -q -rA > $O/test_multigpu_n4.log 2>&1
echo "multigpu rc $?" >> $O/test_multigpu_n4.log
T4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631"
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632"
B4="timeout 600 $T4 bench.py --gpus 4 --steps 50 --warmup 5"
B2="timeout 600 $T2 bench.py --gpus 2 --steps 50 --warmup 5"
$B4 > $O/bench_n4_int8.log 2>&1
for M in fp16 topk qsgd fp8; do $B4 --no-e2e --method $M > $O/bench_n4_$M.log 2>&1; done
$B4 --no-e2e --gpus-per-cluster 2 --workload ernie-m-large-adapters > $O/bench_n4_2x2_int8.log 2>&1
$B4 --no-e2e --gpus-per-cluster 2 --workload ernie-m-large-adapters --method topk > $O/bench_n4_2x2_topk.log 2>&1
$B4 --no-e2e --gpus-per-cluster 4 --workload ernie-m-large-adapters > $O/bench_n4_1x4_int8.log 2>&1
$B2 > $O/bench_n2_int8.log 2>&1
for M in fp16 topk qsgd; do $B2 --no-e2e --method $M > $O/bench_n2_$M.log 2>&1; done
timeout 900 $T4 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > $O/bench_n4_reference.log 2>&1
