# Round 2: two-phase row kernels vs the current default (C4 first 256
# iterations, C2, C1, C5 at K = 1024).
mkdir -p gpurun_out/s5
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for v in cur tp4c4 tp4c3 tp8c2; do
  if [ "$v" = cur ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/ab/libbatchlp_cuda_$v.so; fi
  echo "=== $v"
  timeout 300 python scripts/window_profile.py c4 0,8,64,256 2>&1 | tail -4
  timeout 300 python scripts/run_config.py c2 2 2>&1 | grep "c2:" | tail -1
  timeout 300 python scripts/run_config.py c1 2 2>&1 | grep "c1:" | tail -1
  timeout 300 python scripts/run_config.py c5 1 2>&1 | grep "c5:\|primal\|dual" | tail -3
done > gpurun_out/s5/tp.log 2>&1
cat gpurun_out/s5/tp.log
