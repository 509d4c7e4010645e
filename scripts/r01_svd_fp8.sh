timeout 600 python -m pytest tests/test_gpu_svd.py -m gpu -x -q > gpurun_out/svd_tests.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp8 or FP8 or dense_parity or nonfinite or decompress_single" > gpurun_out/fp8_tests.log 2>&1
timeout 300 python scripts/bench_svd.py > gpurun_out/bench_svd.log 2>&1
timeout 300 python bench.py --method fp8 --no-cpu --no-e2e --steps 50 > gpurun_out/bench_fp8.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/svd_launches.csv python scripts/bench_svd.py --rhos 0.6 --iters 2 --warmup 1 > gpurun_out/svd_ncu.log 2>&1
