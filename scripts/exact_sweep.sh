# exact-path cap sweep on config 1-B&B (one wave)
for cfg in "4096 4" "2048 4" "2048 8" "8192 4" "1024 8" "4096 2" "1024 4" "512 8"; do
  set -- $cfg
  echo "== cap0 $1 growth $2"
  OSERVE_EXACT_CAP0=$1 OSERVE_EXACT_GROWTH=$2 OSERVE_DEBUG_EXACT=1 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "frontier|phaseA round|top replay|phaseB|gpu exhaustive" | tail -9
done
