# exact-path sweep on config 1-B&B: deep split of small late rounds (max new tasks x levels)
python -m pytest tests/test_gpu_exact.py -q -x 2>&1 | tail -1
for cfg in "0 1" "30000 1" "100000 1" "100000 2"; do
  set -- $cfg
  echo "== deep $1 levels $2"
  OSERVE_EXACT_DEEP=$1 OSERVE_EXACT_DEEP_LEVELS=$2 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "gpu exhaustive" | tail -1
done
OSERVE_DEBUG_EXACT=1 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "^\[exact\] [a-zA-Z]" | tail -9
OSERVE_EXACT_DEEP=30000 python -m pytest tests/test_gpu_exact.py -q -x 2>&1 | tail -1
OSERVE_EXACT_DEEP=30000 OSERVE_DEBUG_EXACT=1 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "^\[exact\] [a-zA-Z]" | tail -9
