# A/B of one environment knob on the C4 full-width window (first 64 iterations).
# usage: bash scripts/r02/gpu_env_ab.sh out_dir VAR v1 v2 ...   ("-" = unset)
out=gpurun_out/$1; var=$2; shift 2
mkdir -p $out
for v in "$@"; do
  if [ "$v" = - ]; then unset $var; else export $var=$v; fi
  echo "=== $var=$v"
  MAXIT=${MAXIT:-64} timeout 300 python scripts/run_config.py ${CFG:-c4} 2 > $out/$v.log 2>&1
  grep -A12 "^${CFG:-c4}:" $out/$v.log | tail -13 | grep "^c\|primal \|dual "
done 2>&1 | tee $out/ab.log
