mkdir -p gpurun_out
: > gpurun_out/tt2.log
timeout 300 python scripts/run_config.py c1 2 >> gpurun_out/tt2.log 2>&1
timeout 300 python scripts/run_config.py c2 2 >> gpurun_out/tt2.log 2>&1
grep "us/pass=\|tail_" gpurun_out/tt2.log
timeout 300 python scripts/window_profile.py c2 512,640,1024,100000 2>&1 | tail -5
timeout 1500 python -m pytest tests -x -q -m gpu -k "${PYTEST_K:-core or cpp}" > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
