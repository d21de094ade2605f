# Slice-staged kernels: parity + window timing with/without (run under gpurun).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_core.py -x -q -m gpu -k "slice or loop" > gpurun_out/pytest_core.log 2>&1
tail -3 gpurun_out/pytest_core.log
W=scripts/window_profile.py
timeout 300 python $W c2 64,256,512,1024 > gpurun_out/win_slice.log 2>&1
BATCHLP_SLICE_CH=64 timeout 300 python $W c2 64,256 >> gpurun_out/win_slice.log 2>&1
BATCHLP_SLICE_CH=96 timeout 300 python $W c2 64,256 >> gpurun_out/win_slice.log 2>&1
BATCHLP_NO_SLICE=1 timeout 300 python $W c2 64,256,512,1024 >> gpurun_out/win_slice.log 2>&1
cat gpurun_out/win_slice.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_slice.log 2>&1
tail -1 gpurun_out/bench_slice.log | cut -c1-400
