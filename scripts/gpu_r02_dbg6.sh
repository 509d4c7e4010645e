#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 600 python scripts/dbg_topk_stress.py 0.1 30 > gpurun_out/dbg6_10.log 2>&1; echo "rc $?" >> gpurun_out/dbg6_10.log
timeout 600 python scripts/dbg_topk_stress.py 0.01 30 > gpurun_out/dbg6_1.log 2>&1; echo "rc $?" >> gpurun_out/dbg6_1.log
timeout 600 python scripts/dbg_topk_stress.py 0.1 30 > gpurun_out/dbg6_10b.log 2>&1; echo "rc $?" >> gpurun_out/dbg6_10b.log
