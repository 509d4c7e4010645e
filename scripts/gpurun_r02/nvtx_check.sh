#!/bin/bash
# 1 GPU: NVTX ranges around the public stage calls — parity subset, smoke, default bench.
mkdir -p gpurun_out/nvtx
O=gpurun_out/nvtx
python -m paper_2205_09470_b200.build > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_self.py -q -x -k "fused_step or topk_parity or self_push or self_pull or hierarchical" > $O/tests.log 2>&1; echo "rc $?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 600 python bench.py --no-cpu > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --no-cpu --no-e2e --method topk > $O/bench_topk1.json 2>> $O/bench_default.err
