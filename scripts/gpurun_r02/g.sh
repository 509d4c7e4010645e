#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_self.py -x -q -k "topk" > gpurun_out/topk_tests.log 2>&1
echo "topk rc $?" >> gpurun_out/topk_tests.log
timeout 300 python bench.py --method topk --no-cpu --no-e2e --steps 50 > gpurun_out/bench_topk1.log 2>&1
timeout 300 python bench.py --method topk --density 0.1 --no-cpu --no-e2e --steps 30 > gpurun_out/bench_topk10.log 2>&1
rm -f gpurun_out/sweep_topk_big.jsonl
timeout 900 python scripts/sweep.py --config 5 --sizes 24,28 --out gpurun_out/sweep_topk_big.jsonl > gpurun_out/sweep_topk_big.log 2>&1
