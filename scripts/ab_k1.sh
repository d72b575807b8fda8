# A/B two K1 builds (build/<a>, build/<b>) on config 5 and 5-7B, alternating
a=$1; b=$2
for r in 1 2 3; do
for v in $a $b; do
  for c in cfg5 cfg5_7b; do
    OSERVE_GPU_LIB=build/$v/liboserve_gpu.so timeout 300 python scripts/k1_time.py $c 5 2>&1 | tail -1
  done
done; done
