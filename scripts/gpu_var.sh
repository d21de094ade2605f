# A/B of library variants vs main on C2 windows and C1/C5 (run under gpurun).
mkdir -p gpurun_out
: > gpurun_out/var.log
for v in main $VARIANTS; do
  if [ $v = main ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/variants/libbatchlp_cuda_$v.so; fi
  echo "== $v" >> gpurun_out/var.log
  timeout 300 python scripts/window_profile.py c2 256,512,640,1024,100000 >> gpurun_out/var.log 2>&1
  timeout 300 python scripts/run_config.py c1 2 2>&1 | grep "us/pass=" >> gpurun_out/var.log
  MAXIT=256 timeout 300 python scripts/run_config.py c5 1 2>&1 | grep "us/pass=" >> gpurun_out/var.log
done
cat gpurun_out/var.log
