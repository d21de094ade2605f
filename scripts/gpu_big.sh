mkdir -p gpurun_out
timeout 900 python scripts/run_config.py c4 1 > gpurun_out/run_c4.log 2>&1
timeout 600 python scripts/run_config.py c3 1 > gpurun_out/run_c3.log 2>&1
timeout 600 python scripts/run_config.py c5 1 > gpurun_out/run_c5.log 2>&1
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
cat gpurun_out/run_c4.log gpurun_out/run_c3.log gpurun_out/run_c5.log
tail -1 gpurun_out/bench_c3.log | cut -c1-400
