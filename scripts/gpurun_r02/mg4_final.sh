#!/bin/bash
# final 4-GPU pass of round 2 on the final tree: multi-process parity (2x1, 1x2, 4x1, 2x2, 1x4),
# bench at N = 4 (FP16 fused step over pull, top-k push policy, the copy-engine intra hop),
# config 5 for top-k after the multi-CTA resolve.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests/test_multigpu.py -q -rA > gpurun_out/test_multigpu_n4_final.log 2>&1
echo "multigpu rc $?" >> gpurun_out/test_multigpu_n4_final.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631"
B="timeout 600 $TR bench.py --gpus 4 --steps 50 --warmup 5"
$B > gpurun_out/bench_n4f_int8.log 2>&1
$B --no-e2e --method fp16 > gpurun_out/bench_n4f_fp16.log 2>&1
$B --no-e2e --method topk > gpurun_out/bench_n4f_topk.log 2>&1
$B --no-e2e --method topk --exchange pull > gpurun_out/bench_n4f_topk_pull.log 2>&1
$B --no-e2e --method topk --exchange nccl > gpurun_out/bench_n4f_topk_nccl.log 2>&1
$B --no-e2e --gpus-per-cluster 2 --workload ernie-m-large-adapters > gpurun_out/bench_n4f_2x2_int8.log 2>&1
$B --no-e2e --gpus-per-cluster 2 --workload ernie-m-large-adapters --intra p2p-ce > gpurun_out/bench_n4f_2x2_int8_ce.log 2>&1
$B --no-e2e --gpus-per-cluster 2 --workload ernie-m-large-adapters --intra nccl > gpurun_out/bench_n4f_2x2_int8_nccl.log 2>&1
$B --no-e2e --gpus-per-cluster 4 --workload ernie-m-large-adapters > gpurun_out/bench_n4f_1x4_int8.log 2>&1
rm -f gpurun_out/config5_n4_final.jsonl
timeout 900 $TR scripts/sweep.py --config 5 --sizes 22,26,28 --out gpurun_out/config5_n4_final.jsonl > gpurun_out/sweep_c5_n4f.log 2>&1
