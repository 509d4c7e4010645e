timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "qsgd" > gpurun_out/qsgd_tests.log 2>&1
timeout 300 python bench.py --method qsgd --no-cpu --no-e2e --steps 50 > gpurun_out/bench_qsgd.log 2>&1
