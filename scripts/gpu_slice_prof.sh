# ncu capture of the slice kernels (host-stepped loop so launches are visible).
mkdir -p gpurun_out
export BATCHLP_LOOP=step MAXIT=40
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_slice" -s 10 -c 2 -o gpurun_out/prof_slice python scripts/run_config.py c2 1 > gpurun_out/ncu_slice.log 2>&1
BATCHLP_NO_SLICE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 10 -c 2 -o gpurun_out/prof_noslice python scripts/run_config.py c2 1 >> gpurun_out/ncu_slice.log 2>&1
tail -5 gpurun_out/ncu_slice.log
ls -la gpurun_out
