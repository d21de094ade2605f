# Round profile set (run under gpurun): launch list + traffic of the dominant
# kernels over one C2 solve (host-stepped launches so ncu sees every kernel),
# and ncu --set full captures of k_primal / k_dual at C2 and C5.
mkdir -p gpurun_out
export BATCHLP_LOOP=step
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2_r1.csv python scripts/run_config.py c2 1 > gpurun_out/ncu_list.log 2>&1
MAXIT=40 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 6 -c 2 -o gpurun_out/full_c2_r1 python scripts/run_config.py c2 1 > gpurun_out/ncu_c2.log 2>&1
MAXIT=40 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 6 -c 2 -o gpurun_out/full_c5_r1 python scripts/run_config.py c5 1 > gpurun_out/ncu_c5.log 2>&1
unset BATCHLP_LOOP
BATCHLP_LOOP=cluster MAXIT=300 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tail_fast" -c 1 -o gpurun_out/full_tail_r1 python scripts/run_config.py c1 1 > gpurun_out/ncu_tail.log 2>&1
ls -la gpurun_out
