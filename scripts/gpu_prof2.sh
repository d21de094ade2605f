mkdir -p gpurun_out
W=scripts/window_profile.py
for v in d4 d2; do BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/variants/libbatchlp_cuda_$v.so timeout 300 python $W c5 64 >> gpurun_out/win_var.log 2>&1; BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/variants/libbatchlp_cuda_$v.so timeout 300 python $W c2 64,256 >> gpurun_out/win_var.log 2>&1; done
cat gpurun_out/win_var.log
export BATCHLP_LOOP=step
MAXIT=40 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 6 -c 2 -o gpurun_out/prof_c5_r2 python scripts/run_config.py c5 1 > gpurun_out/ncu_c5.log 2>&1
MAXIT=40 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 6 -c 2 -o gpurun_out/prof_c2_r2 python scripts/run_config.py c2 1 > gpurun_out/ncu_c2.log 2>&1
ls -la gpurun_out
