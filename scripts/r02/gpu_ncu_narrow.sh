# ncu --set full of the narrow single-block passes in the C4 tail (<= 4 LPs).
mkdir -p gpurun_out/nar
export BATCHLP_LOOP=step
MAXIT=6000 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)_narrow" -s 3000 -c 2 -o gpurun_out/nar/narrow_c4 python scripts/run_config.py c4 1 > gpurun_out/nar/ncu.log 2>&1
tail -3 gpurun_out/nar/ncu.log
