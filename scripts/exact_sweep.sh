# exact-path sweep on config 1-B&B: first cap x growth x rounds
for cfg in "8192 4 6" "8192 2 10" "8192 1 12" "4096 2 10" "16384 1 10" "4096 1 14" "8192 3 8" "2048 2 12"; do
  set -- $cfg
  echo "== cap0 $1 growth $2 rounds $3"
  OSERVE_EXACT_CAP0=$1 OSERVE_EXACT_GROWTH=$2 OSERVE_EXACT_ROUNDS=$3 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "gpu exhaustive" | tail -1
done
