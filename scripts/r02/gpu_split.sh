# Round 2: narrow passes as separate kernels (IF(narrow) graph branches), the
# out-of-line residual fold, and the dual at 3 CTAs/SM (spill-free).
mkdir -p gpurun_out/sp
timeout 1500 python -m pytest tests/test_gpu_core.py tests/test_gpu_regressions.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/sp/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/sp/pytest.log
for v in cur dual3; do
  if [ "$v" = cur ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/ab/libbatchlp_cuda_$v.so; fi
  echo "=== $v"
  for r in 1 2; do timeout 300 python scripts/run_config.py c4 2 2>&1 | grep "c4:\|primal\|dual \|decide" | tail -4; done
  timeout 300 python scripts/run_config.py c2 3 2>&1 | grep "c2:" | tail -1
  timeout 300 python scripts/run_config.py c5 2 2>&1 | grep "c5:" | tail -1
  timeout 300 python scripts/run_config.py c3 2 2>&1 | grep "c3:" | tail -1
  timeout 300 python scripts/run_config.py c1 2 2>&1 | grep "c1:" | tail -1
done
