# Round 2: folded residuals (decide) + standalone SpMM geometry.
mkdir -p gpurun_out/s7
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s7/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/s7/pytest_gpu.log
BATCHLP_TAIL_TRACE=1 timeout 600 python scripts/window_profile.py c2 0,64,256,512,1024,100000 > gpurun_out/s7/win_c2.log 2>&1; grep -v "tail trace\]" gpurun_out/s7/win_c2.log | tail -40
timeout 300 python scripts/run_config.py c2 3 2>&1 | grep "c2:"
timeout 300 python scripts/run_config.py c4 2 2>&1 | grep "c4:\|primal\|dual \|decide"
timeout 900 python scripts/c5_sweep.py --out gpurun_out/s7/c5_sweep > gpurun_out/s7/c5_sweep.log 2>&1; tail -16 gpurun_out/s7/c5_sweep.log
