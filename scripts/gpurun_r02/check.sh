#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fallback or structured or topk_parity" > gpurun_out/check_tests.log 2>&1
echo "rc $?" >> gpurun_out/check_tests.log
