mkdir -p gpurun_out
BATCHLP_TAIL_TRACE=1 MAXIT=64 timeout 300 python scripts/run_config.py c2 1 > gpurun_out/tt.log 2>&1
BATCHLP_TAIL_TRACE=1 MAXIT=256 timeout 300 python scripts/run_config.py c2 1 >> gpurun_out/tt.log 2>&1
BATCHLP_TAIL_TRACE=1 MAXIT=64 timeout 300 python scripts/run_config.py c5 1 >> gpurun_out/tt.log 2>&1
cat gpurun_out/tt.log
