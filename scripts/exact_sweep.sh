# exact-path: frontier target with the 1,024 x 2 caps
for tg in 4096 1024 256 64; do
  echo "== target $tg"
  OSERVE_EXACT_TARGET=$tg timeout 200 python scripts/time_exact.py 2>&1 | grep -E "gpu exhaustive" | tail -1
  OSERVE_EXACT_TARGET=$tg OSERVE_DEBUG_EXACT=1 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "^\[exact\] [a-zA-Z]" | tail -8
done
for cfg in "512 2" "1024 3" "256 2"; do set -- $cfg; echo "== cap0 $1 growth $2 target 1024"
  OSERVE_EXACT_TARGET=1024 OSERVE_EXACT_CAP0=$1 OSERVE_EXACT_GROWTH=$2 OSERVE_EXACT_ROUNDS=16 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "gpu exhaustive" | tail -1
done
