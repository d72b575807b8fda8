# exact-path sweep on config 1-B&B: first cap x growth x frontier target
for cfg in "8192 4 0" "8192 2 0" "4096 2 0" "16384 2 0" "8192 3 0" "8192 4 16384" "8192 2 16384" "4096 4 16384" "2048 4 32768"; do
  set -- $cfg
  echo "== cap0 $1 growth $2 target $3"
  OSERVE_EXACT_CAP0=$1 OSERVE_EXACT_GROWTH=$2 OSERVE_EXACT_TARGET=$3 OSERVE_EXACT_ROUNDS=10 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "gpu exhaustive" | tail -1
done
