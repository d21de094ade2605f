mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
W=scripts/window_profile.py
for t in 1 0; do
BATCHLP_TMA=$t timeout 300 python $W c2 64,256,512 >> gpurun_out/win_tma.log 2>&1
BATCHLP_TMA=$t timeout 300 python $W c5 64 >> gpurun_out/win_tma.log 2>&1
BATCHLP_TMA=$t timeout 300 python $W c3 64 >> gpurun_out/win_tma.log 2>&1
done
cat gpurun_out/win_tma.log
