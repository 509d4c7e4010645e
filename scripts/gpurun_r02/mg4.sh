#!/bin/bash
# 4-GPU pass: multi-process parity (every P x G split that fits: 2x1, 1x2, 4x1, 2x2, 1x4),
# bench at N = 4 (every codec; config 3 as 2 clusters x 2 GPUs; config 4), config 5 sweep at N = 4.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests/test_multigpu.py -q -rA > gpurun_out/test_multigpu_n4.log 2>&1
echo "multigpu rc $?" >> gpurun_out/test_multigpu_n4.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621"
B="timeout 600 $TR bench.py --gpus 4 --steps 50 --warmup 5"
$B > gpurun_out/bench_n4_int8.log 2>&1
$B --no-e2e --method fp16 > gpurun_out/bench_n4_fp16.log 2>&1
$B --no-e2e --method topk > gpurun_out/bench_n4_topk.log 2>&1
$B --no-e2e --method fp8 > gpurun_out/bench_n4_fp8.log 2>&1
$B --no-e2e --method fp8e5m2 > gpurun_out/bench_n4_e5m2.log 2>&1
$B --no-e2e --method qsgd > gpurun_out/bench_n4_qsgd.log 2>&1
$B --no-e2e --workload transformer-big > gpurun_out/bench_n4_tbig_int8.log 2>&1
$B --no-e2e --gpus-per-cluster 2 --workload ernie-m-large-adapters > gpurun_out/bench_n4_2x2_adapters_int8.log 2>&1
$B --no-e2e --gpus-per-cluster 2 --workload ernie-m-large-adapters --exact-scale > gpurun_out/bench_n4_2x2_adapters_int8_xscale.log 2>&1
$B --no-e2e --gpus-per-cluster 2 --workload ernie-m-large-adapters --method topk > gpurun_out/bench_n4_2x2_adapters_topk.log 2>&1
rm -f gpurun_out/config5_n4.jsonl
timeout 900 $TR scripts/sweep.py --config 5 --sizes 20,24,26,28 --out gpurun_out/config5_n4.jsonl > gpurun_out/sweep_c5_n4.log 2>&1
