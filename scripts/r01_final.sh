python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_n1.log 2>&1
timeout 300 python bench.py --method fp8 --no-cpu --no-e2e --steps 100 > gpurun_out/bench_fp8.log 2>&1
timeout 300 python scripts/bench_svd.py > gpurun_out/bench_svd.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/svd_launches.csv python scripts/bench_svd.py --rhos 0.6 --iters 2 --warmup 1 > gpurun_out/svd_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk or decompress_single or smoke or fp8_fused" > gpurun_out/topk_tests.log 2>&1
timeout 300 python bench.py --method topk --no-cpu --no-e2e --steps 50 > gpurun_out/bench_topk.log 2>&1
