# Round 2 final validation on HEAD: every GPU test, smoke, the C4 bench line
# (+ reference arm), C2 line, launch list of a short host-stepped C4 run.
mkdir -p gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/fin/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin/smoke.log
timeout 1200 python bench.py --steps 3 --warmup 3 --record-iterations > gpurun_out/fin/bench_c4.json 2> gpurun_out/fin/bench_c4.err; echo "bench rc=$?"; cat gpurun_out/fin/bench_c4.json
cp profiles/gpu_iterations.json gpurun_out/fin/
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fin/bench_c4_ref.json 2>&1; echo "ref rc=$?"; cat gpurun_out/fin/bench_c4_ref.json
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/fin/bench_c2.json 2> gpurun_out/fin/bench_c2.err; echo "c2 rc=$?"; cat gpurun_out/fin/bench_c2.json
BATCHLP_LOOP=step MAXIT=70 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/launches_c4_step.csv python scripts/run_config.py c4 1 > gpurun_out/fin/ncu_list.log 2>&1; gzip -f gpurun_out/fin/launches_c4_step.csv; tail -3 gpurun_out/fin/ncu_list.log
