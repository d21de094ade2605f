# Round 2: A/B of the staged row kernels (cp.async streamed operands, deep
# gathers, occupancy) on C4 (first 256 iterations), C2 and C1.
mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for v in base dyn0 pol0 nar0 lazy fc0; do
  export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/ab/libbatchlp_cuda_$v.so
  echo "=== $v"
  timeout 300 python scripts/window_profile.py c4 0,8,64,256 2>&1 | tail -4
  timeout 300 python scripts/run_config.py c2 2 2>&1 | grep "c2:" | tail -1
  timeout 300 python scripts/run_config.py c1 1 2>&1 | grep "c1:" | tail -1
done > gpurun_out/s3/variants.log 2>&1
cat gpurun_out/s3/variants.log

