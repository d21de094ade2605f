# Standard GPU pass (run under gpurun): tests, smoke, window profiles, bench, traces.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -1 gpurun_out/smoke.log
W=scripts/window_profile.py
timeout 300 python $W c2 64,256,512,1024,100000 > gpurun_out/win.log 2>&1
timeout 300 python $W c5 64 >> gpurun_out/win.log 2>&1
timeout 300 python $W c3 64 >> gpurun_out/win.log 2>&1
timeout 300 python $W c1 100000 >> gpurun_out/win.log 2>&1
cat gpurun_out/win.log
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1
tail -1 gpurun_out/bench_c2.log | cut -c1-300
BATCHLP_TAIL_TRACE=1 MAXIT=64 timeout 300 python scripts/run_config.py c2 1 > gpurun_out/tt.log 2>&1
BATCHLP_TAIL_TRACE=1 timeout 300 python scripts/run_config.py c2 1 >> gpurun_out/tt.log 2>&1
cat gpurun_out/tt.log
BATCHLP_TAIL_TRACE=1 MAXIT=64 timeout 300 python scripts/run_config.py c2 1 > gpurun_out/tt.log 2>&1
BATCHLP_TAIL_TRACE=1 MAXIT=256 timeout 300 python scripts/run_config.py c2 1 >> gpurun_out/tt.log 2>&1
BATCHLP_TAIL_TRACE=1 MAXIT=64 timeout 300 python scripts/run_config.py c5 1 >> gpurun_out/tt.log 2>&1
cat gpurun_out/tt.log
