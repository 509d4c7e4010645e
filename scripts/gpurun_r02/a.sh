#!/bin/bash
# round-2 GPU pass: build, the SELF-transport tests (every P2P path on one GPU), then the suite
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_self.py -x -q > gpurun_out/self_tests.log 2>&1
echo "self rc $?" >> gpurun_out/self_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_self.py > gpurun_out/gpu_tests.log 2>&1
echo "suite rc $?" >> gpurun_out/gpu_tests.log
