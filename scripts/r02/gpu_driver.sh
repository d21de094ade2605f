# The driver's own commands on HEAD (round-end shape): the bench at its
# default config with --steps 20 --warmup 5, then the reference arm.
mkdir -p gpurun_out/drv
/usr/bin/time -v timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv/bench.json 2> gpurun_out/drv/bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/drv/bench.json; grep "Elapsed" gpurun_out/drv/bench.err
/usr/bin/time -v timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv/ref.json 2> gpurun_out/drv/ref.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/drv/ref.json; grep "Elapsed" gpurun_out/drv/ref.err
