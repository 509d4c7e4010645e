#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "qsgd or no_error_feedback or int8_kernels" > gpurun_out/qsgd_tests.log 2>&1
echo "rc $?" >> gpurun_out/qsgd_tests.log
timeout 300 python bench.py --method qsgd --no-cpu --no-e2e --steps 50 > gpurun_out/bench_qsgd.log 2>&1
timeout 300 python bench.py --method int8 --no-ef --no-cpu --no-e2e --steps 50 > gpurun_out/bench_int8_noef.log 2>&1
timeout 300 python bench.py --method fp8e5m2 --no-cpu --no-e2e --steps 50 > gpurun_out/bench_e5m2.log 2>&1
