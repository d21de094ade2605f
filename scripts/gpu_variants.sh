# A/B of library variants and L2 budgets (run under gpurun).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for v in v1 c2 c3 c4; do
  for l2 in 8 16 32; do
    export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/variants/libbatchlp_cuda_$v.so
    export BATCHLP_L2_BUDGET_MB=$l2
    echo "== $v l2=$l2" >> gpurun_out/variants.log
    MAXIT=512 timeout 300 python scripts/run_config.py c2 1 >> gpurun_out/variants.log 2>&1
    MAXIT=128 timeout 300 python scripts/run_config.py c5 1 >> gpurun_out/variants.log 2>&1
    MAXIT=128 timeout 300 python scripts/run_config.py c3 1 >> gpurun_out/variants.log 2>&1
    [ $v = v1 ] && break
  done
done
