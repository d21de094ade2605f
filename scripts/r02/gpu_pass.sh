# Round 2: fused per-block pass (k_pass) vs separate kernels.
mkdir -p gpurun_out/p1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_core.py tests/test_gpu_fullsize.py tests/test_gpu_regressions.py -m gpu -x -q > gpurun_out/p1/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/p1/pytest.log
for v in pass nopass; do
  if [ "$v" = nopass ]; then export BATCHLP_NO_PASS=1; else unset BATCHLP_NO_PASS; fi
  echo "=== $v"
  timeout 300 python scripts/run_config.py c4 2 2>&1 | grep "c4:\|primal\|dual \|pass \|decide" | tail -5
  timeout 300 python scripts/run_config.py c3 2 2>&1 | grep "c3:" | tail -1
  timeout 300 python scripts/run_config.py c5 2 2>&1 | grep "c5:" | tail -1
done
unset BATCHLP_NO_PASS
export BATCHLP_LOOP=step
MAXIT=12 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pass" -s 4 -c 1 -o gpurun_out/p1/full_c4_pass python scripts/run_config.py c4 1 > gpurun_out/p1/ncu.log 2>&1; tail -2 gpurun_out/p1/ncu.log
