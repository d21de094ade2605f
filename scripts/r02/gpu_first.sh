# Round-2 first GPU pass on the restored HEAD: GPU tests, smoke, the C4
# bench line (recording per-LP iterations for the reference arm), the
# reference arm, then the C4 window profile and ncu captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1500 python bench.py --steps 3 --warmup 3 --record-iterations > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_c4.json; tail -5 gpurun_out/bench_c4.err
cp profiles/gpu_iterations.json gpurun_out/ 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_c4_ref.json 2> gpurun_out/bench_c4_ref.err; echo "ref rc=$?"
tail -c 2000 gpurun_out/bench_c4_ref.json; tail -3 gpurun_out/bench_c4_ref.err
bash scripts/r02/gpu_c4_probe.sh
