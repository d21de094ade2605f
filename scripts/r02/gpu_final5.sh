# Round 2 (session 3) validation after the context-grid change.
mkdir -p gpurun_out/f5
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f5/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/f5/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f5/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f5/smoke.log
timeout 1200 python bench.py --steps 3 --warmup 3 --record-iterations > gpurun_out/f5/bench_c4.json 2> gpurun_out/f5/bench_c4.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/f5/bench_c4.json
cp profiles/gpu_iterations.json gpurun_out/f5/
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f5/bench_c4_ref.json 2>&1; echo "ref rc=$?"; cut -c1-200 gpurun_out/f5/bench_c4_ref.json
for c in c2 c1 c3 c5; do timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/f5/bench_$c.json 2> gpurun_out/f5/bench_$c.err; echo "$c rc=$?"; cut -c1-160 gpurun_out/f5/bench_$c.json; done
timeout 900 python scripts/window_profile.py c4 0,8,64,256,1024,2048,4096,100000 > gpurun_out/f5/win_c4.log 2>&1
timeout 1200 python scripts/c5_sweep.py --out gpurun_out/f5/c5_sweep > gpurun_out/f5/c5_sweep.log 2>&1; echo "sweep rc=$?"; tail -15 gpurun_out/f5/c5_sweep.log
export BATCHLP_LOOP=step
MAXIT=12 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 10 -c 2 -o gpurun_out/f5/full_c4 python scripts/run_config.py c4 1 > gpurun_out/f5/ncu_c4.log 2>&1; tail -1 gpurun_out/f5/ncu_c4.log
MAXIT=70 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f5/launches_c4_step.csv python scripts/run_config.py c4 1 > gpurun_out/f5/ncu_list.log 2>&1; gzip -f gpurun_out/f5/launches_c4_step.csv; echo done
