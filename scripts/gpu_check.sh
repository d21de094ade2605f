# Standard GPU pass (run under gpurun): tests, smoke, sweeps, bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -1 gpurun_out/smoke.log
for c in c2; do timeout 600 python scripts/phase_sweep.py $c auto > gpurun_out/sweep_$c.log 2>&1; done
for tb in 1 2 4; do for cl in 8 16; do echo "== tail_blocks=$tb cluster=$cl" >> gpurun_out/tail.log; BATCHLP_TAIL_BLOCKS=$tb BATCHLP_TAIL_CLUSTER=$cl timeout 300 python scripts/run_config.py c2 2 >> gpurun_out/tail.log 2>&1; done; done
MAXIT=128 timeout 300 python scripts/run_config.py c5 1 > gpurun_out/run_c5.log 2>&1
MAXIT=128 timeout 300 python scripts/run_config.py c3 1 > gpurun_out/run_c3.log 2>&1
