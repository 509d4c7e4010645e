timeout 600 python -m pytest tests/test_gpu_svd.py -m gpu -x -q > gpurun_out/svd_tests3.log 2>&1
timeout 300 python scripts/bench_svd.py --rhos 0.9,0.6,0.2 > gpurun_out/bench_svd_simt.log 2>&1
timeout 300 python scripts/bench_svd.py --rhos 0.6 --gram dmma > gpurun_out/bench_svd_dmma.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/svd_launches2.csv python scripts/bench_svd.py --rhos 0.6 --iters 2 --warmup 1 > gpurun_out/svd_ncu2.log 2>&1
