for a in "--method identity" "--method fp16" "--method topk --density 0.1" "--method topk --density 0.1 --values i8" "--method topk --density 0.01 --values f16" "--method int8 --no-ef" "--method fp8" "--method qsgd"; do
  timeout 300 python bench.py $a --no-cpu --no-e2e --steps 50 >> gpurun_out/codecs_n1.log 2>&1
done
