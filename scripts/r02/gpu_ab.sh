# A/B of library variants (lib/ab/libbatchlp_cuda_<tag>.so vs the main
# build "cur"): C4 at full width (first 64 iterations), then whole solves.
# usage: bash scripts/r02/gpu_ab.sh out_dir tag1 [tag2 ...]   (AB_FULL=1: whole solves too)
out=gpurun_out/$1; shift
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for v in cur "$@"; do
  if [ "$v" = cur ]; then unset BATCHLP_LIB; else export BATCHLP_LIB=$PWD/paper_2601_21990_b200/lib/ab/libbatchlp_cuda_$v.so; fi
  echo "=== $v"
  MAXIT=64 timeout 300 python scripts/run_config.py c4 2 > $out/$v.c4w.log 2>&1
  grep -A12 "c4:" $out/$v.c4w.log | tail -13 | grep "c4:\|primal \|dual "
  if [ -n "$AB_FULL" ]; then
    for c in c4 c2 c5 c3 c1; do
      timeout 300 python scripts/run_config.py $c 2 > $out/$v.$c.log 2>&1
      grep "^$c:" $out/$v.$c.log | tail -1
    done
  fi
done 2>&1 | tee $out/ab.log
