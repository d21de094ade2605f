# Round 2: dual register-pressure variants (inline division in all; late
# streams, no narrow dispatch, 3 CTAs/SM) on a full C4 solve, C2, C1; then
# the core GPU tests on the default build.
mkdir -p gpurun_out/s6
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for v in cur late nar0 dual3 latenar0; do
  if [ "$v" = cur ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/ab/libbatchlp_cuda_$v.so; fi
  echo "=== $v"
  timeout 300 python scripts/run_config.py c4 1 2>&1 | grep "c4:\|primal\|dual \|decide\|check"
  timeout 300 python scripts/run_config.py c2 2 2>&1 | grep "c2:" | tail -1
  timeout 300 python scripts/run_config.py c1 2 2>&1 | grep "c1:" | tail -1
done > gpurun_out/s6/div.log 2>&1
cat gpurun_out/s6/div.log
unset BATCHLP_LIB
timeout 900 python -m pytest tests/test_gpu_core.py tests/test_mps_tools.py tests/test_gpu_regressions.py -m gpu -x -q > gpurun_out/s6/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/s6/pytest.log
