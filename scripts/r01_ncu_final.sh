python scripts/profile_step.py --method int8 --steps 3 > gpurun_out/ncu_plain_run.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_int8_ws -s 1 -c 1 -o gpurun_out/int8_step_final python scripts/profile_step.py --method int8 --steps 3 > gpurun_out/ncu_final.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_final.log 2>&1
