# exact path: parity tests + timing (config 1-B&B) with per-phase laps
timeout 300 python -m pytest tests/test_gpu_exact.py -q -x 2>&1 | tail -25
timeout 200 python scripts/time_exact.py 2>&1 | tail -5
OSERVE_DEBUG_EXACT=1 timeout 200 python scripts/time_exact.py 2>&1 | grep -E "^\[exact\] [a-zA-Z]" | tail -8
