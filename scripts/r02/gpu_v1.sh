# Round 2: one slot per lane (a warp per row) for W = 32, with 4- or 8-deep
# gather batches, vs the two-slot lanes.
mkdir -p gpurun_out/v1s
for v in v1 v1b8 v1p8; do
  export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/ab/libbatchlp_cuda_$v.so
  timeout 600 python -m pytest tests/test_gpu_core.py -m gpu -x -q 2>&1 | tail -1
done
for v in cur v1 v1b8 v1p8; do
  if [ "$v" = cur ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/ab/libbatchlp_cuda_$v.so; fi
  echo "=== $v"
  timeout 300 python scripts/run_config.py c4 2 2>&1 | grep "c4:\|primal\|dual \|decide" | tail -4
  timeout 300 python scripts/run_config.py c2 3 2>&1 | grep "c2:" | tail -1
  timeout 300 python scripts/run_config.py c5 2 2>&1 | grep "c5:" | tail -1
  timeout 300 python scripts/run_config.py c3 2 2>&1 | grep "c3:" | tail -1
  timeout 300 python scripts/run_config.py c1 2 2>&1 | grep "c1:" | tail -1
done
