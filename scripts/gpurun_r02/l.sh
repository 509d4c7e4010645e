#!/bin/bash
# 1 GPU: the TMA-ring top-k stage pass (parity + bench vs plain loads), the serialized top-k
# phase breakdown (no two-stream pipeline) at 1 % and 10 %, and ncu of the INT8 fused step
# without EF (DRAM bytes vs algorithmic: is g re-read from HBM?).
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "topk" > gpurun_out/topk_tests.log 2>&1
echo "topk rc $?" >> gpurun_out/topk_tests.log
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 30"
for D in 0.01 0.1; do
  $B --method topk --density $D > gpurun_out/bench_topk_${D}_tma.log 2>&1
  $B --method topk --density $D --topk-stage plain > gpurun_out/bench_topk_${D}_plain.log 2>&1
  $B --method topk --density $D --no-pipeline > gpurun_out/bench_topk_${D}_tma_nopipe.log 2>&1
  $B --method topk --density $D --no-pipeline --topk-stage plain > gpurun_out/bench_topk_${D}_plain_nopipe.log 2>&1
done
$B --method int8 --no-ef > gpurun_out/bench_int8_noef.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_int8_ws -s 2 -c 1 -o gpurun_out/ncu_noef \
  python scripts/profile_step.py --method int8 --no-ef --steps 3 > gpurun_out/ncu_noef.log 2>&1
ncu -i gpurun_out/ncu_noef.ncu-rep --page raw --csv > gpurun_out/ncu_noef_raw.csv 2>&1
rm -f gpurun_out/ncu_noef.ncu-rep
