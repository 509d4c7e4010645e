#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "topk or decompress_single" > gpurun_out/topk_tests.log 2>&1
echo "topk rc $?" >> gpurun_out/topk_tests.log
timeout 300 python bench.py --method topk --no-cpu --no-e2e --steps 50 > gpurun_out/bench_topk1.log 2>&1
timeout 300 python bench.py --method topk --density 0.1 --no-cpu --no-e2e --steps 30 > gpurun_out/bench_topk10.log 2>&1
timeout 300 python bench.py --method topk --density 0.1 --values i8 --no-cpu --no-e2e --steps 30 > gpurun_out/bench_topk10_i8.log 2>&1
