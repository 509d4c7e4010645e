timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -x -q > gpurun_out/mg_tests2.log 2>&1
for args in "--gpus 4 --workload transformer-big --method fp8" "--gpus 4 --workload transformer-big --method qsgd" "--gpus 4 --gpus-per-cluster 4 --workload ernie-m-large-adapters" "--gpus 4 --workload ernie-m-base"; do
  n=$(echo $args | awk '{print $2}')
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 bench.py $args --steps 50 --warmup 5 --no-e2e --no-cpu >> gpurun_out/mg_bench2.log 2>&1
done
