timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -x -q -k "2-1 or 4-1" > gpurun_out/mg_tests3.log 2>&1
for m in fp8 qsgd; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --workload transformer-big --method $m --steps 50 --warmup 5 --no-e2e --no-cpu >> gpurun_out/mg_bench3.log 2>&1
done
