for r in 1 2; do
for v in base m4_2 m4_3; do
  echo "== $v"; OSERVE_GPU_LIB=build/$v/liboserve_gpu.so timeout 300 python scripts/k1_time.py cfg5_7b 5 2>&1 | tail -1
done; done
