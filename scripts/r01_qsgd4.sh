timeout 300 python bench.py --method qsgd --no-cpu --no-e2e --steps 50 > gpurun_out/bench_qsgd_c0.log 2>&1
timeout 300 python bench.py --method qsgd --no-cpu --no-e2e --steps 50 --step-config 1 > gpurun_out/bench_qsgd_c1.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "qsgd_kernels" > gpurun_out/qsgd_tests4.log 2>&1
