timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_svd.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/gpu_tests3.log 2>&1
timeout 300 python bench.py --method qsgd --no-cpu --no-e2e --steps 50 > gpurun_out/bench_qsgd.log 2>&1
