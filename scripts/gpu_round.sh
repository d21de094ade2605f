# Standard pass (run under gpurun): GPU tests, smoke, windows, bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -1 gpurun_out/smoke.log
timeout 300 python scripts/window_profile.py c2 64,256,512,1024,100000 > gpurun_out/win.log 2>&1
timeout 300 python scripts/window_profile.py c1 100000 >> gpurun_out/win.log 2>&1
cat gpurun_out/win.log
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1
tail -1 gpurun_out/bench_c2.log > gpurun_out/bench_c2.json
python -c "import json; d=json.load(open('gpurun_out/bench_c2.json')); print(d['value'], d['e2e'], json.dumps(d['roofline'])[:700])"
