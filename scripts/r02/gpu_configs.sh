# Round 2: bench lines for every BASELINE config (C1-C5; C4 is the default
# line, C5 at K=1024) with the reference timed beside them.
mkdir -p gpurun_out/cfg
for c in c1 c3 c5; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 3 > gpurun_out/cfg/bench_$c.json 2> gpurun_out/cfg/bench_$c.err; echo "$c rc=$?"
  tail -c 600 gpurun_out/cfg/bench_$c.json
done
# the reference arm on C1 (full convergence) and C3 (time-boxed, extrapolated)
timeout 900 python bench.py --impl reference --config c1 --steps 2 --warmup 3 > gpurun_out/cfg/bench_c1_ref.json 2>&1; tail -c 400 gpurun_out/cfg/bench_c1_ref.json
