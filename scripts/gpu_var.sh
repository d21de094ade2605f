# A/B of one library variant vs main on the tail-heavy configs (run under gpurun).
mkdir -p gpurun_out
: > gpurun_out/var.log
for v in main $VARIANTS; do
  if [ $v = main ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/variants/libbatchlp_cuda_$v.so; fi
  echo "== $v" >> gpurun_out/var.log
  timeout 300 python scripts/run_config.py c1 2 >> gpurun_out/var.log 2>&1
  timeout 300 python scripts/run_config.py c2 2 >> gpurun_out/var.log 2>&1
done
grep "==\|us/pass=\|tail_" gpurun_out/var.log
