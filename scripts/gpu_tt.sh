mkdir -p gpurun_out
BATCHLP_TAIL_TRACE=1 timeout 300 python scripts/run_config.py c2 1 > gpurun_out/tt.log 2>&1
BATCHLP_TAIL_TRACE=1 timeout 300 python scripts/run_config.py c1 1 >> gpurun_out/tt.log 2>&1
cat gpurun_out/tt.log
