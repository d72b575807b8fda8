# exact-path: frontier target per plan (debug laps)
for tg in 4096 8192 16384; do
  echo "== target $tg"
  OSERVE_EXACT_TARGET=$tg timeout 200 python scripts/time_exact.py 2>&1 | grep -E "gpu exhaustive" | tail -1
  OSERVE_EXACT_TARGET=$tg OSERVE_DEBUG_EXACT=1 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "^\[exact\] [a-zA-Z]" | tail -9
done
