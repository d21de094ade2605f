# Round 2: prefetched row metadata (pipelined walk) vs the plain walk.
mkdir -p gpurun_out/pf
timeout 900 python -m pytest tests/test_gpu_core.py tests/test_gpu_regressions.py -m gpu -x -q > gpurun_out/pf/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pf/pytest.log
for v in cur pf0 pf1c3; do
  if [ "$v" = cur ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/ab/libbatchlp_cuda_$v.so; fi
  echo "=== $v"
  timeout 300 python scripts/run_config.py c4 2 2>&1 | grep "c4:\|primal\|dual \|decide" | tail -4
  timeout 300 python scripts/run_config.py c2 2 2>&1 | grep "c2:" | tail -1
  timeout 300 python scripts/run_config.py c5 2 2>&1 | grep "c5:" | tail -1
  timeout 300 python scripts/run_config.py c3 2 2>&1 | grep "c3:" | tail -1
done
