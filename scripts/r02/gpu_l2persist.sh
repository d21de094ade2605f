# L2 set-aside for persisting (evict_last) gathers: C4 per-launch primal/dual
# at K=1024 (first 64 iterations) vs the set-aside size.
mkdir -p gpurun_out/l2p
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for mb in none 16 32 64 96 200; do
  if [ "$mb" = none ]; then unset BATCHLP_L2_PERSIST_MB; else export BATCHLP_L2_PERSIST_MB=$mb; fi
  echo "=== persist $mb"
  MAXIT=64 timeout 300 python scripts/run_config.py c4 2 2>&1 | grep -v "^ *\(compact\|check\)" | tail -5
done 2>&1 | tee gpurun_out/l2p/c4.log
