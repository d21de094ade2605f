# Round 2 (session 3) validation after the narrow-pass occupancy change.
mkdir -p gpurun_out/f4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f4/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/f4/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f4/smoke.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/f4/bench_c4.json 2> gpurun_out/f4/bench_c4.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/f4/bench_c4.json
for c in c3 c5 c2 c1; do timeout 1200 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/f4/bench_$c.json 2> gpurun_out/f4/bench_$c.err; echo "$c rc=$?"; cut -c1-160 gpurun_out/f4/bench_$c.json; done
timeout 900 python scripts/window_profile.py c4 0,8,64,256,1024,2048,4096,100000 > gpurun_out/f4/win_c4.log 2>&1; cat gpurun_out/f4/win_c4.log
