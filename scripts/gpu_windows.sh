mkdir -p gpurun_out
W=scripts/window_profile.py
timeout 300 python $W c2 64,256,512,1024,100000 > gpurun_out/win.log 2>&1
BATCHLP_LOOP=graph timeout 300 python $W c2 64,256,512,1024 >> gpurun_out/win.log 2>&1
BATCHLP_TAIL_BLOCKS=4 timeout 300 python $W c2 64,256,512,1024,100000 >> gpurun_out/win.log 2>&1
BATCHLP_TAIL_BLOCKS=16 timeout 300 python $W c2 64,256,512,1024,100000 >> gpurun_out/win.log 2>&1
timeout 300 python $W c5 64,128 >> gpurun_out/win.log 2>&1
timeout 300 python $W c3 64,128 >> gpurun_out/win.log 2>&1
timeout 300 python $W c1 64,100000 >> gpurun_out/win.log 2>&1
cat gpurun_out/win.log
