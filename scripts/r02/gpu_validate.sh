# Round 2 validation on HEAD: every GPU test, smoke, the C4 bench line
# (recording per-LP iterations for the reference arm) and the reference arm,
# the C2 line, the C5 batch-size sweep, and the C4 ncu launch list + a full
# capture of k_primal / k_dual at K = 1024.
mkdir -p gpurun_out/v1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v1/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/v1/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/v1/smoke.log
timeout 1200 python bench.py --steps 3 --warmup 3 --record-iterations > gpurun_out/v1/bench_c4.json 2> gpurun_out/v1/bench_c4.err; echo "bench rc=$?"; cat gpurun_out/v1/bench_c4.json; tail -3 gpurun_out/v1/bench_c4.err
cp profiles/gpu_iterations.json gpurun_out/v1/
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/v1/bench_c4_ref.json 2>&1; echo "ref rc=$?"; cat gpurun_out/v1/bench_c4_ref.json
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/v1/bench_c2.json 2> gpurun_out/v1/bench_c2.err; echo "c2 rc=$?"; cat gpurun_out/v1/bench_c2.json
BATCHLP_TAIL_TRACE=1 timeout 600 python scripts/window_profile.py c2 0,64,256,512,1024,100000 > gpurun_out/v1/win_c2.log 2>&1; tail -30 gpurun_out/v1/win_c2.log
timeout 600 python scripts/window_profile.py c4 0,8,64,256,1024,2048,4096,100000 > gpurun_out/v1/win_c4.log 2>&1; cat gpurun_out/v1/win_c4.log
timeout 1500 python scripts/c5_sweep.py --out gpurun_out/v1/c5_sweep > gpurun_out/v1/c5_sweep.log 2>&1; echo "sweep rc=$?"; tail -20 gpurun_out/v1/c5_sweep.log
export BATCHLP_LOOP=step
MAXIT=12 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(primal|dual)" -s 10 -c 2 -o gpurun_out/v1/full_c4 python scripts/run_config.py c4 1 > gpurun_out/v1/ncu_c4.log 2>&1; tail -2 gpurun_out/v1/ncu_c4.log
unset BATCHLP_LOOP
MAXIT=300 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v1/launches_c4.csv python scripts/run_config.py c4 1 > gpurun_out/v1/ncu_list_c4.log 2>&1; gzip -f gpurun_out/v1/launches_c4.csv; ls -la gpurun_out/v1
