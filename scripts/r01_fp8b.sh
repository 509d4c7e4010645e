timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp8 or FP8" > gpurun_out/fp8_tests.log 2>&1
timeout 300 python bench.py --method fp8 --no-cpu --no-e2e --steps 50 > gpurun_out/bench_fp8.log 2>&1
