# Profiling pass (run under gpurun). Host-stepped loop (BATCHLP_LOOP=step) so
# ncu sees individual launches (graph kernel nodes behind conditional nodes
# cannot be profiled).
mkdir -p gpurun_out
export BATCHLP_LOOP=step
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python scripts/run_config.py c2 1 > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 20 -c 4 -o gpurun_out/prof_c2 python scripts/run_config.py c2 1 > gpurun_out/ncu_full_c2.log 2>&1
MAXIT=32 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 20 -c 4 -o gpurun_out/prof_c5 python scripts/run_config.py c5 1 > gpurun_out/ncu_full_c5.log 2>&1
ls -la gpurun_out
