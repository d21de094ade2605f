mkdir -p gpurun_out
B=scripts/microbench/_build/gather_bench
timeout 300 $B 20000 40000 10 1024 > gpurun_out/micro_c5_primal.log 2>&1
timeout 300 $B 40000 20000 20 1024 > gpurun_out/micro_c5_dual.log 2>&1
timeout 300 $B 2000 2000 10 4000 > gpurun_out/micro_c2.log 2>&1
timeout 300 $B 100000 200000 10 1024 > gpurun_out/micro_c4.log 2>&1
cat gpurun_out/micro_*.log
