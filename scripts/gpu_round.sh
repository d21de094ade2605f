set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1
for c in c1 c3 c5; do timeout 600 python scripts/run_config.py $c 2 > gpurun_out/run_$c.log 2>&1; done
tail -5 gpurun_out/*.log
