timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/topk_launches.csv python bench.py --method topk --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/topk_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_topk_(densify|resolve|bracket|merge|scan|move)" -s 20 -c 8 -o gpurun_out/topk_full python bench.py --method topk --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/topk_full.log 2>&1
timeout 600 python -m pytest tests/test_gpu_svd.py -m gpu -x -q > gpurun_out/svd_tests2.log 2>&1
timeout 300 python scripts/bench_svd.py --eig syevj --rhos 0.9,0.6,0.2 > gpurun_out/bench_svd_syevj.log 2>&1
