# Round 2: A/B of the staged row kernels (cp.async streamed operands, deep
# gathers, occupancy) on C4 (first 256 iterations), C2 and C1.
mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for v in default d4 nostage d8c3 d4c3; do
  if [ "$v" = default ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/variants/libbatchlp_cuda_$v.so; fi
  echo "=== $v"
  timeout 300 python scripts/window_profile.py c4 0,8,64,256 2>&1 | tail -4
  timeout 300 python scripts/run_config.py c2 2 2>&1 | grep "c2:" | tail -1
  timeout 300 python scripts/run_config.py c1 1 2>&1 | grep "c1:" | tail -1
done > gpurun_out/s3/variants.log 2>&1
cat gpurun_out/s3/variants.log
unset BATCHLP_LIB
timeout 900 python -m pytest tests/test_mps_tools.py tests/test_gpu_core.py -m gpu -x -q > gpurun_out/s3/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/s3/pytest.log
