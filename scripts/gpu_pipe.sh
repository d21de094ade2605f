# A/B of gather-pipeline / occupancy variants on the bulk windows (run under gpurun).
mkdir -p gpurun_out
W=scripts/window_profile.py
: > gpurun_out/pipe.log
for v in main pipe pipe3 base3; do
  if [ $v = main ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/variants/libbatchlp_cuda_$v.so; fi
  echo "== $v" >> gpurun_out/pipe.log
  timeout 300 python $W c2 64,256,512 >> gpurun_out/pipe.log 2>&1
  timeout 300 python $W c5 64 >> gpurun_out/pipe.log 2>&1
  timeout 300 python $W c3 64 >> gpurun_out/pipe.log 2>&1
done
cat gpurun_out/pipe.log
