#!/bin/bash
# Final 1-GPU pass of round 2: full GPU suite, smoke, the default bench line (with the CPU
# baseline and e2e), every codec's line, the reference arm, and the ncu launch list of the
# default bench command plus a full capture of the top-k 1 % kernels.
mkdir -p gpurun_out/final_n1
O=gpurun_out/final_n1
python -m paper_2205_09470_b200.build > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 50"
for M in fp16 identity fp8 fp8e5m2 qsgd; do $B --method $M > $O/bench_$M.json 2>> $O/bench_err.log; done
$B --no-ef > $O/bench_int8_noef.json 2>> $O/bench_err.log
$B --method topk > $O/bench_topk1.json 2>> $O/bench_err.log
$B --method topk --density 0.1 > $O/bench_topk10.json 2>> $O/bench_err.log
$B --method topk --values i8 > $O/bench_topk1_i8.json 2>> $O/bench_err.log
$B --method topk --density 0.1 --values i8 > $O/bench_topk10_i8.json 2>> $O/bench_err.log
$B --workload transformer-big > $O/bench_tbig.json 2>> $O/bench_err.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_default.csv \
  python bench.py --steps 2 --warmup 3 > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_topk_(stage|densify|merge|resolve|move)" -c 6 --csv --page raw \
  python scripts/profile_step.py --method topk --steps 2 > $O/ncu_topk1_raw.csv 2> $O/ncu_topk1.err
