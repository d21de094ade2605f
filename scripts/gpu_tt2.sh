mkdir -p gpurun_out
BATCHLP_TAIL_TRACE=1 timeout 300 python scripts/run_config.py c2 1 > gpurun_out/tt2.log 2>&1
timeout 300 python scripts/run_config.py c1 2 >> gpurun_out/tt2.log 2>&1
timeout 300 python scripts/run_config.py c2 2 >> gpurun_out/tt2.log 2>&1
grep "trace\]\|fast decide\|us/pass=" gpurun_out/tt2.log | grep -v "decide trace"
timeout 1200 python -m pytest tests -x -q -m gpu -k "core or cpp" > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
