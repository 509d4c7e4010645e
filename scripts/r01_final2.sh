python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_n1.log 2>&1
timeout 300 python bench.py --method topk --no-cpu --no-e2e --steps 50 > gpurun_out/bench_topk.log 2>&1
