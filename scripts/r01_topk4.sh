timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk or decompress_single or smoke or fp8_fused" > gpurun_out/topk_tests.log 2>&1
timeout 300 python bench.py --method topk --no-cpu --no-e2e --steps 50 > gpurun_out/bench_topk.log 2>&1
