#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python tests/debug_topk_race.py 109432384 6 > gpurun_out/dbg5_race.log 2>&1
echo "rc $?" >> gpurun_out/dbg5_race.log
