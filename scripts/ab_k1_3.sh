for r in 1 2; do for v in base2 fin; do for c in cfg5 cfg5_7b cfg2; do
  OSERVE_GPU_LIB=build/$v/liboserve_gpu.so timeout 300 python scripts/k1_time.py $c 5 2>&1 | tail -1
done; done; done
