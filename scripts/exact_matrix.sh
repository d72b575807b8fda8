for cfg in "1 1 0 0" "1 0 0 0" "0 1 0 0" "1 1 1 0" "0 0 1 0" "0 0 0 0" "0 0 0 1" "1 1 0 1" "0 0 1 1"; do
  set -- $cfg
  echo "== LEAFFLAG=$1 LBM=$2 PHASE_L=$3 REPLAY=$4"
  OSERVE_EXACT_LEAFFLAG=$1 OSERVE_EXACT_LBM=$2 OSERVE_EXACT_PHASE_L=$3 OSERVE_EXACT_REPLAY=$4 timeout 300 python -m pytest tests/test_gpu_exact.py -q 2>&1 | tail -1
done
