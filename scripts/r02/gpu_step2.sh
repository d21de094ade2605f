# Round 2, second GPU pass: the new parity / boundary / sharding / MPS tests,
# then the C4 window profile and ncu captures after dynamic work items, the
# gather L2 policy and narrow single-block rows; C2 decide trace.
mkdir -p gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_cpp.py tests/test_mps_tools.py tests/test_gpu_core.py tests/test_gpu_regressions.py -m gpu -x -q > gpurun_out/s2/pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/s2/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/s2/smoke.log
timeout 600 python scripts/window_profile.py c4 0,8,64,256,1024,2048,4096,100000 > gpurun_out/s2/win_c4.log 2>&1; cat gpurun_out/s2/win_c4.log
BATCHLP_TAIL_TRACE=1 timeout 300 python scripts/window_profile.py c2 0,64,256,512,1024,100000 > gpurun_out/s2/win_c2.log 2>&1; cat gpurun_out/s2/win_c2.log
export BATCHLP_LOOP=step
MAXIT=12 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 10 -c 2 -o gpurun_out/s2/full_c4 python scripts/run_config.py c4 1 > gpurun_out/s2/ncu_c4.log 2>&1
tail -2 gpurun_out/s2/ncu_c4.log
ls -la gpurun_out/s2
