#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_self.py -x -q > gpurun_out/self_tests.log 2>&1
echo "self rc $?" >> gpurun_out/self_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "e5m2 or E5M2 or pull_reducer or dense_parity" > gpurun_out/e5m2_tests.log 2>&1
echo "e5m2 rc $?" >> gpurun_out/e5m2_tests.log
