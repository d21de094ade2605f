mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/tail_profile.py c2 1024 >> gpurun_out/tail_prof.log 2>&1
BATCHLP_NO_FAST_TAIL=1 timeout 300 python scripts/tail_profile.py c2 1024 >> gpurun_out/tail_prof.log 2>&1
BATCHLP_TAIL_CLUSTER=8 timeout 300 python scripts/tail_profile.py c2 1024 >> gpurun_out/tail_prof.log 2>&1
BATCHLP_TAIL_BLOCKS=4 timeout 300 python scripts/tail_profile.py c2 256 >> gpurun_out/tail_prof.log 2>&1
timeout 300 python scripts/tail_profile.py c1 1 >> gpurun_out/tail_prof.log 2>&1
cat gpurun_out/tail_prof.log
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1
tail -1 gpurun_out/bench_c2.log
