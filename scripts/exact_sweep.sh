# exact-path sweep on config 1-B&B: first phase-A round run a warp per task
python -m pytest tests/test_gpu_exact.py -q -x 2>&1 | tail -1
for w in 99 1 2 0; do
  echo "== warp from round $w"
  OSERVE_EXACT_WARP_FROM=$w timeout 200 python scripts/time_exact.py 2>&1 | grep -E "gpu exhaustive" | tail -1
done
OSERVE_DEBUG_EXACT=1 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "^\[exact\] [a-zA-Z]" | tail -9
