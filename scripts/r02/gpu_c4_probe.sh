# Round-2 first look at the north-star config C4 (K=1024, m=100k, n=200k):
# window profile, then ncu --set full of k_primal / k_dual at full width and
# a launch list of the first 300 iterations with DRAM traffic per launch.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python scripts/window_profile.py c4 0,8,64,256,512,1024,2048,4096,100000 > gpurun_out/win_c4.log 2>&1
cat gpurun_out/win_c4.log
export BATCHLP_LOOP=step
MAXIT=12 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 10 -c 2 -o gpurun_out/full_c4_k1024 python scripts/run_config.py c4 1 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
MAXIT=1200 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python scripts/run_config.py c4 1 > gpurun_out/ncu_list_c4.log 2>&1
tail -3 gpurun_out/ncu_list_c4.log
gzip -f gpurun_out/launches_c4.csv
ls -la gpurun_out
