# exact-path check: B&B parity tests, then config 1-B&B timings over the wave count
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for W in 1 3 6; do
  echo "== WAVES=$W"
  OSERVE_EXACT_WAVES=$W timeout 300 python -m pytest tests/test_gpu_exact.py -q 2>&1 | tail -1
  OSERVE_EXACT_WAVES=$W OSERVE_DEBUG_EXACT=1 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "frontier|phaseA round|wave check|top replay|phaseB|gpu exhaustive|reference" | tail -22
done
