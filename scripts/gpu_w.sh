mkdir -p gpurun_out
W=scripts/window_profile.py
for mw in 16 32; do
BATCHLP_MAX_W=$mw timeout 300 python $W c2 64,256,512,1024,100000 >> gpurun_out/win_w.log 2>&1
BATCHLP_MAX_W=$mw timeout 300 python $W c5 64 >> gpurun_out/win_w.log 2>&1
BATCHLP_MAX_W=$mw timeout 300 python $W c3 64 >> gpurun_out/win_w.log 2>&1
done
cat gpurun_out/win_w.log
