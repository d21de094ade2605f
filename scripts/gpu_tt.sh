# Tail phase trace (full C2 and C1 solves) + core GPU tests + bench (run under gpurun).
mkdir -p gpurun_out
BATCHLP_TAIL_TRACE=1 timeout 300 python scripts/run_config.py c2 1 > gpurun_out/tt.log 2>&1
BATCHLP_TAIL_TRACE=1 timeout 300 python scripts/run_config.py c1 1 >> gpurun_out/tt.log 2>&1
timeout 300 python scripts/run_config.py c2 2 >> gpurun_out/tt.log 2>&1
timeout 300 python scripts/run_config.py c1 2 >> gpurun_out/tt.log 2>&1
cat gpurun_out/tt.log
timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
[ -n "$NO_BENCH" ] || { timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log | cut -c1-300; }
