timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "qsgd or fp8 or int8_fused or int8_kernels" > gpurun_out/qsgd_tests.log 2>&1
timeout 300 python bench.py --method qsgd --no-cpu --no-e2e --steps 50 > gpurun_out/bench_qsgd.log 2>&1
timeout 300 python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/bench_int8_check.log 2>&1
