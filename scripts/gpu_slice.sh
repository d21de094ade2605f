# Slice kernels: parity + window timing vs the register-gather kernels (run under gpurun).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_core.py -x -q -m gpu -k "slice" > gpurun_out/pytest_core.log 2>&1
tail -3 gpurun_out/pytest_core.log
W=scripts/window_profile.py
: > gpurun_out/win_slice.log
BATCHLP_SLICE=2 timeout 300 python $W c2 64,256,512,1024 >> gpurun_out/win_slice.log 2>&1
BATCHLP_SLICE=2 timeout 300 python $W c1 100000 >> gpurun_out/win_slice.log 2>&1
timeout 300 python $W c2 64,256,512,1024 >> gpurun_out/win_slice.log 2>&1
cat gpurun_out/win_slice.log
export BATCHLP_LOOP=step MAXIT=40 BATCHLP_SLICE=2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_slice" -s 10 -c 2 -o gpurun_out/prof_direct python scripts/run_config.py c2 1 > gpurun_out/ncu_direct.log 2>&1
tail -2 gpurun_out/ncu_direct.log
