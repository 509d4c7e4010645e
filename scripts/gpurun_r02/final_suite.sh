#!/bin/bash
# 1 GPU: the driver's round-end checks on the final tree — pytest -m gpu, smoke, default bench.
mkdir -p gpurun_out/final_suite
O=gpurun_out/final_suite
python -m paper_2205_09470_b200.build > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
